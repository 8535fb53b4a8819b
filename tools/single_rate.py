"""Graph-replayed single-trajectory iteration rate (the bench's C2 / C3 legs).

    python tools/single_rate.py [--configs C2,C3] [--iters 200]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1712_05012_b200 as P  # noqa: E402
from paper_1712_05012_b200 import device as DV  # noqa: E402
from paper_1712_05012_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C2,C3")
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--water", action="store_true")
a = ap.parse_args()
s = DV.stream()
for cfg in a.configs.split(","):
    ch, _, _, fld = workloads.system(cfg, solvation=a.water)
    W, K = 10, a.iters
    r = DV.EnsembleRunner(ch, fld, 1, P.StepConfig(max_iters=W + K, torque_tol_rel=0.0, energy_window=0), chunk=16)
    r.load(workloads.start_theta(cfg, ch)[None, :], np.zeros((1, ch.n_dof), bool))
    r.prepare(W)
    r.prepare(K)
    with torch.cuda.stream(s):
        r.run_graph(W)
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        r.run_graph(K)
        e1.record(s)
    s.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{cfg}: {ch.n_atoms} atoms, {K / (ms * 1e-3):.0f} it/s, {ms / K * 1e3:.1f} us/iteration", flush=True)
