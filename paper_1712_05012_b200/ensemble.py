"""Trajectory-parallel ensembles across GPUs.

One chain does not shard (iteration t+1 needs every force of t and the step
normalises by the global max |tau|, kcm.py:270-273), but independent
trajectories do.  Trajectory r goes to rank floor(r * G / B) — contiguous
blocks — and every rank replays the same host RNG stream, so starts match
``kinefold fold --init random --batch B --seed S`` exactly (cli.py:136,
:146-147).  There is no communication per iteration; one collective at the
end gathers each trajectory's record (final theta, last energies, tau_max,
iteration count, stop reason) to rank 0 — an all-gather over NCCL (NVLink /
NVSwitch) with the ``nccl`` backend, or gloo on CPU for the tests.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

REASON_CODES = {"max_iters": 1, "torque-free": 2, "torque tolerance": 3,
                "torque tolerance (relative)": 4, "energy plateau": 5}
CODE_REASONS = {v: k for k, v in REASON_CODES.items()}


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard(total: int, rank: int, size: int) -> tuple[int, int]:
    """Contiguous block of trajectories owned by `rank`: r -> floor(r*G/B)."""
    lo = -(-rank * total // size)
    hi = -(-(rank + 1) * total // size)
    return lo, hi


def owner(r: int, total: int, size: int) -> int:
    return r * size // total


def gather_rows(local: torch.Tensor, total: int, rank: int, size: int, group=None) -> torch.Tensor | None:
    """All-gather per-rank row blocks [B_local, ...] into [total, ...] (rank 0 keeps it)."""
    if size == 1:
        return local
    width = max(hi - lo for lo, hi in (shard(total, k, size) for k in range(size)))
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(size)]
    dist.all_gather(parts, pad, group=group)
    if rank != 0:
        return None
    rows = [parts[k][:hi - lo] for k, (lo, hi) in enumerate(shard(total, k, size) for k in range(size))]
    return torch.cat(rows, dim=0)


def pack_result(res) -> dict:
    """Per-trajectory end-of-run record of an EnsembleResult (host arrays)."""
    B = len(res.iterations)
    last = np.zeros((B, 4))
    for k in range(B):
        if res.iterations[k] > 0:
            last[k] = res.energies[k, res.iterations[k] - 1]
    return dict(theta=np.asarray(res.theta, float), last=last,
                iterations=np.asarray(res.iterations, np.int64),
                reason=np.array([REASON_CODES.get(r, 0) for r in res.reasons], np.int64))


def gather_records(rec: dict, total: int, device=None, group=None) -> dict | None:
    rank, size = world()
    out = {}
    for key, arr in rec.items():
        t = torch.as_tensor(arr)
        if device is not None:
            t = t.to(device)
        g = gather_rows(t, total, rank, size, group)
        if g is not None:
            out[key] = g.cpu().numpy()
    return out if rank == 0 else None


def run_sharded(chain, fld, thetas_all: np.ndarray, step, frozen=None, device=None, group=None):
    """Run this rank's block of trajectories on its GPU, gather to rank 0.

    Returns (gathered records on rank 0 else None, local EnsembleResult).
    """
    from .device import EnsembleRunner
    rank, size = world()
    total = len(thetas_all)
    lo, hi = shard(total, rank, size)
    runner = EnsembleRunner(chain, fld, hi - lo, step)
    fr = np.zeros((hi - lo, chain.n_dof), bool) if frozen is None else np.asarray(frozen)[lo:hi]
    runner.load(thetas_all[lo:hi], fr)
    runner.run()
    res = runner.result()
    return gather_records(pack_result(res), total, device=device, group=group), res
