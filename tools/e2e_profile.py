"""Breakdown of fold_ensemble's end-to-end time (the bench's e2e leg): runner
lookup, host conformations in, graph replays, results out."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1712_05012_b200 as P  # noqa: E402
from paper_1712_05012_b200 import device as DV  # noqa: E402
from paper_1712_05012_b200 import workloads  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ch, params, w, fld = workloads.system("C2")
th = workloads.random_thetas(ch, 1024, seed=1)
confs = [P.Conformation(t, np.zeros(ch.n_dof, bool), ch.n_residues) for t in th]
step = P.StepConfig(kappa=0.5, max_iters=K, torque_tol_rel=0.0, energy_window=0)
P.fold_ensemble(ch, confs, fld, step)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    dc = DV.device_chain(ch)
    df = DV.device_field(fld, dc.n_atoms)
    t1 = time.perf_counter()
    runner = [v for (_, _, v) in DV._runner_cache._d.values()][-1]
    runner.load([c.theta for c in confs], [c.frozen for c in confs])
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    runner.run()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    res = runner.result()
    t4 = time.perf_counter()
    print(f"tables {1e3*(t1-t0):.2f}  load {1e3*(t2-t1):.2f}  run {1e3*(t3-t2):.2f}  result {1e3*(t4-t3):.2f} ms")
    t0 = time.perf_counter()
    P.fold_ensemble(ch, confs, fld, step)
    t5 = time.perf_counter()
    print(f"  fold_ensemble {1e3*(t5-t0):.2f} ms -> {1024*K/(t5-t0):,.0f} traj-it/s")
