import sys, os; sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1712_05012_b200 as P
from paper_1712_05012_b200 import workloads
from oracle import kcm_oracle as O
ch, params, w, fld = workloads.system("C3")
th = workloads.random_thetas(ch, 160, seed=2, angle_range=30.0)
confs = [P.Conformation(t, np.zeros(ch.n_dof, bool), ch.n_residues) for t in th]
st = P.StepConfig(max_iters=1, torque_tol_rel=0.0, energy_window=0)
ens = P.fold_ensemble(ch, confs, fld, st)          # B*n_seg > 592: fk_scan_kernel path
for k in (0, 77, 159):
    pos = P.forward_kinematics(ch, confs[k])        # B=1 path
    _, _, _, ref = O.fk(ch, np.array(th[k]))
    e = fld.evaluate(pos).energy
    print(k, "fk(B=1) vs oracle", np.abs(pos - ref).max(), "ens E", ens.energies[k, 0, :2], "single E", e.g_elec, e.g_vdw,
          "rel", abs(ens.energies[k, 0, 1] - e.g_vdw) / abs(e.g_vdw))
