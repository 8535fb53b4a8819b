"""Small workload for compute-sanitizer (racecheck / memcheck / synccheck):
smoke() plus short ensembles through every pair kernel variant (select with
env: KFB200_CLUSTER_MIN_B=4 puts B=8 on the cluster-pair kernel;
KFB200_CLUSTER=0 with B=32 takes the dense half list) and a water iteration."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402
import paper_1712_05012_b200 as P  # noqa: E402
from paper_1712_05012_b200 import workloads  # noqa: E402

__graft_entry__.smoke()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for water in (False, True):
    ch, params, w, fld = workloads.system("C2", solvation=water)
    th = workloads.random_thetas(ch, B, seed=1)
    confs = [P.Conformation(t, np.zeros(ch.n_dof, bool), ch.n_residues) for t in th]
    res = P.fold_ensemble(ch, confs, fld, P.StepConfig(kappa=0.5, max_iters=2, torque_tol_rel=0.0,
                                                        energy_window=0))
    print("water" if water else "vacuum", "B", B, "iterations", res.iterations.tolist()[:4], flush=True)
print("sanitize case ok")
