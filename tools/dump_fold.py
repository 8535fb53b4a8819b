"""Dump a short ensemble fold (records + final theta) for bitwise A/B of kernel builds.

    python tools/dump_fold.py OUT.npz [--ensemble 256] [--iters 20] [--config C2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1712_05012_b200 as P  # noqa: E402
from paper_1712_05012_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("out")
ap.add_argument("--ensemble", type=int, default=256)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--config", default="C2")
a = ap.parse_args()
ch, params, w, fld = workloads.system(a.config)
th = workloads.random_thetas(ch, a.ensemble, seed=3)
confs = [P.Conformation(t, np.zeros(ch.n_dof, bool), ch.n_residues) for t in th]
res = P.fold_ensemble(ch, confs, fld, P.StepConfig(max_iters=a.iters, torque_tol_rel=0.0, energy_window=0))
np.savez(a.out, energies=res.energies, theta=res.theta)
if len(sys.argv) > 2 and os.path.exists(a.out.replace(".npz", "_ref.npz")):
    pass
print("saved", a.out, res.energies.shape)
