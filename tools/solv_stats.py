"""Solvation enumeration statistics (build with EXTRA=-DSOLV_STATS).

    python tools/solv_stats.py --config C2 --ensemble 64
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1712_05012_b200 as P  # noqa: E402
from paper_1712_05012_b200 import _native as N, device as DV, workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--ensemble", type=int, default=64)
a = ap.parse_args()
ch, params, w, fld = workloads.system(a.config, solvation=True)
th = workloads.random_thetas(ch, a.ensemble, seed=1)
step = P.StepConfig(max_iters=4, torque_tol_rel=0.0, energy_window=0)
r = DV.EnsembleRunner(ch, fld, a.ensemble, step)
r.load(th, np.zeros_like(th, dtype=bool))
lib = N.lib()
fs, bs = N.ref(r.df.struct_for(False)), N.ref(r.batch.struct)
N.check(lib.kf_fk(N.ref(r.dc.struct), bs, DV._sp()), "fk")
N.check(lib.kf_bin(fs, bs, DV._sp()), "bin")
N.check(lib.kf_solvation(fs, bs, DV._sp()), "solv")
out = (C.c_ulonglong * 8)()
lib.kf_debug_solv_stats(out)
g, g2, g1, cand, ex, cr, exg, wsum = list(out)
atoms = a.ensemble * r.df.n_solv_nz
print(f"atoms {atoms}  groups {g} ({g / atoms:.1f}/atom)  settled by 2 full {g2 / g:.1%}  one full {g1 / g:.1%}")
print(f"candidate iterations per unsettled group {cand / max(g - g2, 1):.1f}; mean words {wsum / g:.2f}")
print(f"exposed samples {ex / (32 * g):.2%}, critical {cr / (32 * g):.2%}, groups with exposure {exg / g:.1%}")
