import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1712_05012_b200 as P
from paper_1712_05012_b200 import device as DV, workloads
ch, params, w, fld = workloads.system("C2")
th = workloads.random_thetas(ch, 1024, seed=1)
confs = [P.Conformation(t, np.zeros(ch.n_dof, bool), ch.n_residues) for t in th]
step = P.StepConfig(kappa=0.5, max_iters=50, torque_tol_rel=0.0, energy_window=0)
P.fold_ensemble(ch, confs, fld, step)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    key = (len(confs), repr(step), False, id(fld))
    runner = DV._runner_cache.get(ch, hash(key), lambda: None)
    t1 = time.perf_counter()
    runner.load([c.theta for c in confs], [c.frozen for c in confs])
    torch.cuda.synchronize(); t2 = time.perf_counter()
    runner.run(); torch.cuda.synchronize(); t3 = time.perf_counter()
    res = runner.result(); t4 = time.perf_counter()
    print(f"cache {1e3*(t1-t0):.2f} load {1e3*(t2-t1):.2f} run {1e3*(t3-t2):.2f} result {1e3*(t4-t3):.2f} ms; device-rate run {1024*50/(t3-t2):.0f}")
    t0 = time.perf_counter(); P.fold_ensemble(ch, confs, fld, step); t5 = time.perf_counter()
    print(f"  fold_ensemble total {1e3*(t5-t0):.2f} ms -> {1024*50/(t5-t0):.0f} traj-it/s")
