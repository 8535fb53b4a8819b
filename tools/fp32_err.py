"""fp32 vs fp64 pair-math error on C1/C2 conformations: forces, torques, step.

    python tools/fp32_err.py [package_parent_dir]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else ROOT)
import numpy as np  # noqa: E402

import paper_1712_05012_b200 as P  # noqa: E402
from oracle import kcm_oracle as O  # noqa: E402
from paper_1712_05012_b200 import workloads  # noqa: E402

print(P.__file__, "KFB200_PAIR_F64_BELOW =", os.environ.get("KFB200_PAIR_F64_BELOW", "1 (default)"))
for cfg in ("C1", "C2"):
    ch, params, w, fld = workloads.system(cfg)
    ths = workloads.random_thetas(ch, 3, seed=3) if cfg == "C2" else [workloads.start_theta("C1", ch)]
    for th in ths:
        M, Pp, U, pos = O.fk(ch, th)
        out = {}
        for mode in ("fp32", "fp64"):
            P.set_pair_precision(mode)
            r = fld.evaluate(pos)
            f = np.asarray(r.forces)
            F, T = O.wrenches(ch, pos, f)
            tau = O.torques(ch, U, Pp, F, T)
            out[mode] = (f, r.energy.g_elec + r.energy.g_vdw, tau)
        f32, f64 = out["fp32"][0], out["fp64"][0]
        err = np.abs(f32 - f64).max(1) / np.maximum(np.abs(f64).max(1), 1e-30)
        t32, t64 = out["fp32"][2], out["fp64"][2]
        tmax = np.abs(t64).max()
        dstep = np.abs(t32 / np.abs(t32).max() - t64 / tmax).max()
        print(cfg, "force rel: median %.1e p99 %.1e | energy rel %.1e | tau err/taumax %.1e | step err/kappa %.1e" % (
            np.median(err), np.quantile(err, 0.99), abs(out["fp32"][1] - out["fp64"][1]) / abs(out["fp64"][1]),
            np.abs(t32 - t64).max() / tmax, dstep))
P.set_pair_precision("fp32")
