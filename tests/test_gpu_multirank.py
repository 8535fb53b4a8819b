"""The multi-rank ensemble path executed end to end on the GPU (cli.py:144-169,
`fold --batch`): two ranks share the one B200 of the test box, each folds its
contiguous block of the C5 starts with its own kernels, and the per-trajectory
records are all-gathered (gloo: host-staged, since both ranks are on one GPU).
The gathered records must equal a single-process fold_ensemble of all the
trajectories bit for bit (same kernel decomposition on both sides: B = 8 and
16 both take the small-batch kernels)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOTAL, ITERS = 16, 6


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, size, port, out_q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    import paper_1712_05012_b200 as P
    from paper_1712_05012_b200 import ensemble as ENS
    from paper_1712_05012_b200 import workloads
    ch, params, w, fld = workloads.system("C2")
    thetas = workloads.random_thetas(ch, TOTAL, seed=1)
    step = P.StepConfig(kappa=0.5, max_iters=ITERS, torque_tol_rel=0.0, energy_window=0)
    got, local = ENS.run_sharded(ch, fld, thetas, step)
    lo, hi = ENS.shard(TOTAL, rank, size)
    assert len(local.iterations) == hi - lo
    if rank == 0:
        out_q.put({k: v.tolist() for k, v in got.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_run_sharded_two_ranks_equals_single_process():
    import torch.multiprocessing as mp

    import paper_1712_05012_b200 as P
    from paper_1712_05012_b200 import ensemble as ENS
    from paper_1712_05012_b200 import workloads
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ch, params, w, fld = workloads.system("C2")
    thetas = workloads.random_thetas(ch, TOTAL, seed=1)
    confs = [P.Conformation(t, np.zeros(ch.n_dof, bool), ch.n_residues) for t in thetas]
    ref = ENS.pack_result(P.fold_ensemble(ch, confs, fld, P.StepConfig(kappa=0.5, max_iters=ITERS,
                                                                      torque_tol_rel=0.0, energy_window=0)))
    for key in ("theta", "last", "iterations", "reason"):
        assert np.array_equal(np.asarray(got[key]), ref[key]), key
