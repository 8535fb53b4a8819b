"""Eager KCM iterations of the C5 ensemble (for ncu / per-kernel timing).

    python tools/prof_step.py [--ensemble B] [--iters K] [--water] [--config C2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1712_05012_b200 as P  # noqa: E402
from paper_1712_05012_b200 import _native as N, device as DV, workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ensemble", type=int, default=1024)
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--water", action="store_true")
ap.add_argument("--config", default="C2")
a = ap.parse_args()
ch, params, w, fld = workloads.system(a.config, solvation=a.water)
th = workloads.random_thetas(ch, a.ensemble, seed=1)
step = P.StepConfig(max_iters=a.iters + 1, torque_tol_rel=0.0, energy_window=0)
r = DV.EnsembleRunner(ch, fld, a.ensemble, step)
r.load(th, np.zeros_like(th, dtype=bool))
lib = N.lib()
cs, fs, bs, ss = N.ref(r.dc.struct), N.ref(r.df.struct_for(False)), N.ref(r.batch.struct), N.ref(DV._step_struct(step))
s = DV.stream()
with torch.cuda.stream(s):
    for _ in range(a.iters):
        N.check(lib.kf_fold_iterations_eager(cs, fs, bs, ss, 1, DV._sp()), "iter")
s.synchronize()
st = r.batch.status()
print("ok", a.ensemble, "trajectories,", sum(x.n_pairs for x in st), "pairs, errors", sum(x.error for x in st))
