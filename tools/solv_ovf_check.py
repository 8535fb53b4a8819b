import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1712_05012_b200 as P
from paper_1712_05012_b200 import _native as N, device as DV, workloads
ch, params, w, fld = workloads.system("C3", solvation=True)
th = workloads.random_thetas(ch, 1, seed=1)
step = P.StepConfig(max_iters=30, torque_tol_rel=0.0, energy_window=0)
r = DV.EnsembleRunner(ch, fld, 1, step)
r.load(th, np.zeros_like(th, dtype=bool))
lib = N.lib()
cs, fs, bs = N.ref(r.dc.struct), N.ref(r.df.struct_for(False)), N.ref(r.batch.struct)
N.check(lib.kf_fk(cs, bs, DV._sp()), "fk"); N.check(lib.kf_bin(fs, bs, DV._sp()), "bin")
N.check(lib.kf_solvation(fs, bs, DV._sp()), "solv")
torch.cuda.synchronize()
print("nb_cap", r.batch.struct.nb_cap, "ovf count", int(r.batch.t["solv_ovf"][0]), "status", r.batch.status()[0].error, r.batch.status()[0].overflow)
