"""Multi-rank ensemble plumbing on CPU (gloo, world size 2 and 3): trajectory
sharding, the end-of-run all-gather of per-trajectory records, and the
replayed RNG stream that makes shards match `--init random --batch B`."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1712_05012_b200 import ensemble as ENS
from paper_1712_05012_b200 import workloads


def test_shards_partition_and_owner():
    for total in (1, 7, 1024, 1499):
        for size in (1, 2, 3, 4, 8):
            seen = []
            for rank in range(size):
                lo, hi = ENS.shard(total, rank, size)
                seen += list(range(lo, hi))
                for r in range(lo, hi):
                    assert ENS.owner(r, total, size) == rank
            assert seen == list(range(total))


def test_random_starts_replay_cli_stream():
    """cli.py:136, :146-147: one default_rng(seed), phi then psi per run."""
    import paper_1712_05012_b200 as P
    ch = P.build_chain(["ALA", "SER", "CYS"] * 3)
    th = workloads.random_thetas(ch, 5, seed=7)
    rng = np.random.default_rng(7)
    for r in range(5):
        phi = rng.uniform(-90, 90, ch.n_residues)
        psi = rng.uniform(-90, 90, ch.n_residues)
        assert np.array_equal(th[r], ch.conf_from_backbone(phi, psi).theta)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, size, port, total, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    lo, hi = ENS.shard(total, rank, size)
    # per-trajectory records as a rank would produce them: value = global index
    rec = {"theta": np.arange(lo, hi, dtype=float)[:, None] * np.ones((1, 4)),
           "iterations": np.arange(lo, hi, dtype=np.int64) * 10,
           "reason": np.full(hi - lo, 1, np.int64)}
    got = ENS.gather_records(rec, total)
    if rank == 0:
        out_q.put({k: v.tolist() for k, v in got.items()})
    else:
        assert got is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("size,total", [(2, 1024), (3, 10), (2, 3)])
def test_gather_records_gloo(size, total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, total, q)) for r in range(size)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(np.array(res["theta"])[:, 0], np.arange(total, dtype=float))
    assert res["iterations"] == [10 * r for r in range(total)]
    assert res["reason"] == [1] * total


def test_gather_rows_single_rank_identity():
    t = torch.arange(12.0).reshape(4, 3)
    assert torch.equal(ENS.gather_rows(t, 4, 0, 1), t)
