"""Warm back-to-back time per call of each hot-path entry point (one config, B
trajectories): R calls of the same entry between two events, so launch
overhead overlaps and the number is the kernel's own duration (latency floor).

    python tools/kernel_lat.py --config C2 --ensemble 1
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
ap.add_argument("--config", default="C2")
ap.add_argument("--ensemble", type=int, default=1)
ap.add_argument("--reps", type=int, default=200)
a = ap.parse_args()
ch, params, w, fld = workloads.system(a.config)
th = workloads.random_thetas(ch, a.ensemble, seed=1)
step = P.StepConfig(max_iters=10 ** 6, torque_tol_rel=0.0, energy_window=0)
r = DV.EnsembleRunner(ch, fld, a.ensemble, step)
r.load(th, np.zeros_like(th, dtype=bool))
lib = N.lib()
cs, fs, bs, ss = N.ref(r.dc.struct), N.ref(r.df.struct_for(False)), N.ref(r.batch.struct), N.ref(DV._step_struct(step))
s = DV.stream()
calls = {"fk": lambda: lib.kf_fk(cs, bs, DV._sp()), "bin": lambda: lib.kf_bin(fs, bs, DV._sp()),
         "pairs": lambda: lib.kf_pairs(fs, bs, DV._sp()),
         "torque": lambda: lib.kf_torques_step(cs, fs, bs, ss, DV._sp())}
with torch.cuda.stream(s):
    for f in calls.values():   # one full iteration: valid state for every entry
        N.check(f(), "warm")
    s.synchronize()
    out = {}
    for name, f in calls.items():
        for _ in range(5):
            N.check(f(), name)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0 = lib.kf_launch_counter()
        e0.record(s)
        for _ in range(a.reps):
            N.check(f(), name)
        e1.record(s)
        s.synchronize()
        out[name] = (round(e0.elapsed_time(e1) / a.reps * 1e3, 2), int(lib.kf_launch_counter() - c0) // a.reps)
print(a.config, "B =", a.ensemble, "us per call (kernels per call):", out)
