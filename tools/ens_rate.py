"""C5 ensemble rate (graph-replayed) and the eager pair-phase time, one process.

usage: python tools/ens_rate.py [B] [K]   (env selects kernel variants)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_05012_b200 as P  # noqa: E402
from paper_1712_05012_b200 import _native as N  # noqa: E402
from paper_1712_05012_b200 import device as DV  # noqa: E402
from paper_1712_05012_b200 import workloads  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
K = int(sys.argv[2]) if len(sys.argv) > 2 else 16
water = os.environ.get("WATER") == "1"
ch, params, w, fld = workloads.system("C2", solvation=water)
th = workloads.random_thetas(ch, B, seed=1)
step = P.StepConfig(kappa=0.5, max_iters=3 * K + 8, torque_tol_rel=0.0, energy_window=0)
r = DV.EnsembleRunner(ch, fld, B, step, chunk=8)
r.load(th, np.zeros((B, ch.n_dof), bool))
r.prepare(K)
s = DV.stream()
with torch.cuda.stream(s):
    r.run_graph(K)
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    r.run_graph(K)
    e1.record(s)
    s.synchronize()
ms = e0.elapsed_time(e1) / K
lib = N.lib()
cs, fs, bs = N.ref(r.dc.struct), N.ref(r.df.struct_for(False)), N.ref(r.batch.struct)
ts = []
with torch.cuda.stream(s):
    for _ in range(5):
        a, b_, c_ = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        N.check(lib.kf_fk(cs, bs, DV._sp()), "fk")
        a.record(s)
        N.check(lib.kf_bin(fs, bs, DV._sp()), "bin")
        b_.record(s)
        N.check(lib.kf_pairs(fs, bs, DV._sp()), "pairs")
        c_.record(s)
        s.synchronize()
        ts.append((a.elapsed_time(b_), b_.elapsed_time(c_)))
sa = r.batch.status_array()
bad = int((sa["error"] != 0).sum())
print(f"B={B} env={ {k: v for k, v in os.environ.items() if k.startswith('KFB200')} } "
      f"step {ms:.4f} ms -> {B / ms * 1e3:,.0f} traj-it/s | bin {np.median([t[0] for t in ts]):.4f} ms "
      f"pairs {np.median([t[1] for t in ts]):.4f} ms | P9 {int(sa['n_pairs'].sum())} errors {bad}", flush=True)
