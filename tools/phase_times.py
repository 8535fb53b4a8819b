"""Per-phase CUDA-event times of eager KCM iterations (one config, B trajectories).

    python tools/phase_times.py --config C2 --ensemble 1 [--water]
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
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--water", action="store_true")
a = ap.parse_args()
ch, params, w, fld = workloads.system(a.config, solvation=a.water)
th = workloads.random_thetas(ch, a.ensemble, seed=1)
step = P.StepConfig(max_iters=a.iters + 5, torque_tol_rel=0.0, energy_window=0)
r = DV.EnsembleRunner(ch, fld, a.ensemble, step)
r.load(th, np.zeros_like(th, dtype=bool))
lib = N.lib()
cs, fs, bs, ss = N.ref(r.dc.struct), N.ref(r.df.struct_for(False)), N.ref(r.batch.struct), N.ref(DV._step_struct(step))
s = DV.stream()
names = ["fk", "bin", "pairs", "solv", "torque"]
acc = dict.fromkeys(names, 0.0)
with torch.cuda.stream(s):
    for it in range(a.iters):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record(s)
        N.check(lib.kf_fk(cs, bs, DV._sp()), "fk")
        ev[1].record(s)
        N.check(lib.kf_bin(fs, bs, DV._sp()), "bin")
        ev[2].record(s)
        N.check(lib.kf_pairs(fs, bs, DV._sp()), "pairs")
        ev[3].record(s)
        if a.water:
            N.check(lib.kf_solvation(fs, bs, DV._sp()), "solv")
        ev[4].record(s)
        N.check(lib.kf_torques_step(cs, fs, bs, ss, DV._sp()), "torque")
        ev[5].record(s)
        s.synchronize()
        if it >= 3:
            for k, nm in enumerate(names):
                acc[nm] += ev[k].elapsed_time(ev[k + 1]) / (a.iters - 3)
print(a.config, "B =", a.ensemble, "ms per iteration (eager):", {k: round(v, 4) for k, v in acc.items()},
      "total", round(sum(acc.values()), 4))
