import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np
from conftest import golden, make_system
from oracle import kcm_oracle as O
import paper_1712_05012_b200 as P
g = golden("fold_c1_1000")
ch, params, w, fld = make_system(g["seq"])
conf = P.Conformation(g["theta0"], g["frozen"], ch.n_residues)
for mode in ("fp32", "fp64"):
    P.set_pair_precision(mode)
    tr = P.fold(ch, conf, fld, P.StepConfig(max_iters=1000, torque_tol_rel=0.0, energy_window=0, snapshot_every=0))
    E = np.array([[r.energy.g_elec, r.energy.g_vdw, r.energy.g_cav] for r in tr.records])
    rel = np.abs(E - g["energies"]).sum(1) / np.abs(g["energies"]).sum(1)
    th = np.array([r.theta for r in tr.records])
    for thr in (1e-5, 1e-4, 1e-3):
        idx = np.flatnonzero(rel > thr)
        print(mode, thr, idx[:1], rel.max())
    dth = np.abs(((th[:60] - g["thetas"][:60]) + 180) % 360 - 180).max()
    print(mode, "max dtheta first 60", dth)
    print(mode, "energies at 400, 600, 800, 999", E[[400,600,800,999]].sum(1), g["energies"][[400,600,800,999]].sum(1))
