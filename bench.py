"""Benchmark: KCM iterations/s of the B200 KCM loop (BASELINE.json metric).

Workload: an ensemble of 1024 independent
trajectories of the 140-residue / 1,499-atom synthetic A/C/S chain (C2),
random +-90 starts (`--init random --seed 1 --batch 1024` semantics), vacuum
FieldConfig() defaults, fixed iteration count (torque_tol_rel = 0,
energy_window = 0).  A step is one KCM iteration of every trajectory (FK ->
elec/vdW pair forces -> wrenches -> suffix-scan torques -> max-normalised
step), replayed from CUDA graphs.  With N GPUs (torchrun) every rank folds its
own contiguous block of 1024 trajectories of the one seed-1 start stream
(1024 N in all): trajectories are independent units, so the path partitions
with no data-path collective and the scaling is "weak" (tier rule ⑤); one
NCCL all-gather of the final per-trajectory records ends the timed region.
`--strong` instead splits one 1024-trajectory ensemble over the ranks.

Output: one JSON line on rank 0 (see the README of the driver contract):
value = trajectory-iterations/s of the whole job; e2e = the same through the
public `fold_ensemble` API with host inputs/outputs; roofline of the dominant
kernel; cpu_baseline = the oracle (numpy restatement of the reference,
`oracle/kcm_oracle.py`) timed on this host.  Extra legs on rank 0 at N = 1:
C5 in water (FieldConfig(solvation=True)) with its solvation-coverage rate,
C5 with fp64 pair math (the strict-parity mode), the single-trajectory
configs C1-C4 on the GPU (C3 also through the `fold()` API), and C1 / C3 / C4
on the CPU reference path.

`--impl reference` times the reference CPU algorithm (the oracle port; the
reference is a pure-Python package) on all host cores with a process pool.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

ENSEMBLE = 1024
METRIC = "KCM iterations/sec"
UNIT = "trajectory-iterations/s"
REF_ITERS = 20      # iterations per reference-arm task (one trajectory per core per step)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ensemble", type=int, default=ENSEMBLE, help="trajectories per GPU (weak) or in all (--strong)")
    ap.add_argument("--strong", action="store_true", help="split one ensemble over the ranks (total work fixed)")
    ap.add_argument("--water", action="store_true", help="headline in FieldConfig(solvation=True)")
    ap.add_argument("--no-extras", action="store_true", help="skip the water / fp64 / single-trajectory / CPU legs")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def workload_name(args, water=None) -> str:
    mode = "water" if (args.water if water is None else water) else "vacuum"
    return (f"C5: ensemble of {args.ensemble} x C2 chain (140 random A/C/S residues, 1499 atoms), "
            f"random +-90 starts, {mode}, fixed iterations")


def config_of(args, n_atoms=1499, dofs=518, world=1) -> dict:
    total = args.ensemble if args.strong else args.ensemble * world
    return {"workload": workload_name(args), "ensemble": total, "ensemble_per_gpu": total // max(world, 1),
            "scaling_mode": "strong (one ensemble split over the ranks)" if args.strong else
                            "weak (each rank folds its own 1024-trajectory block of the start stream)",
            "atoms_per_trajectory": n_atoms,
            "dofs": dofs, "parallelism": f"trajectory-parallel x{world}",
            "l2": "working set per step > 126 MB L2 (positions, forces, link transforms of 1.5M atoms / "
                  "530k links), no explicit flush"}


def host_cores() -> dict:
    logical = os.cpu_count() or 1
    physical = logical
    try:
        import psutil
        physical = psutil.cpu_count(logical=False) or logical
    except ImportError:
        pass
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"logical": logical, "physical": physical, "model": model}


# --------------------------------------------------------------------------
# clocks sampled during the timed region
# --------------------------------------------------------------------------

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
            # nvidia-smi takes a moment to start: wait for its first line so that even a
            # short timed region is sampled
            t_end = time.time() + 5.0
            while time.time() < t_end and os.path.getsize(self.path) == 0 and self.proc.poll() is None:
                time.sleep(0.02)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or not f[0].isdigit() or int(f[0]) != self.idx:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:   # no sample in the window: one query right after it
            try:
                q = subprocess.run(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                    f"--id={self.idx}"], capture_output=True, text=True, timeout=30).stdout
                f = [x.strip() for x in q.strip().splitlines()[0].split(",")]
                sm, mx = [float(f[1])], float(f[2])
                reasons = {nm for nm, v in zip(names, f[5:9]) if v.lower() == "active"}
            except (OSError, ValueError, IndexError, subprocess.SubprocessError):
                return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------
# reference arm: the reference CPU algorithm on all host cores
# --------------------------------------------------------------------------

_W = {}


def _ref_init(water: bool):
    """Pool initializer: the C2 system and the oracle field once per worker
    (setup is outside every timed task)."""
    from oracle import kcm_oracle as O
    from paper_1712_05012_b200 import workloads
    _one_thread()   # one process per core: no nested BLAS / OpenMP pools
    ch, params, w, _ = workloads.system("C2")
    _W["ch"], _W["of"] = ch, O.OracleField(params, w, solvation=water)


def _one_thread():
    """Limit numpy's native thread pools to one thread in this process (the
    reference arm runs one process per core; the 1-core leg is one thread)."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except ImportError:
        pass


def _ref_task(theta):
    from oracle import kcm_oracle as O
    ch = _W["ch"]
    O.fold(ch, theta, np.zeros(ch.n_dof, bool), _W["of"], max_iters=REF_ITERS, torque_tol_rel=0.0,
           energy_window=0)
    return REF_ITERS


def reference_arm(args, rank: int):
    import multiprocessing as mp

    from paper_1712_05012_b200 import workloads
    if rank != 0:
        return
    hc = host_cores()
    cores = hc["logical"]
    ch = workloads.system("C2")[0]
    # the bench's own starts: trajectory r of the seed-1 stream, cores of them per step
    thetas = workloads.random_thetas(ch, args.ensemble, seed=1)
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_ref_init, initargs=(args.water,)) as pool:
        pool.map(_ref_task, [thetas[k] for k in range(cores)], chunksize=1)    # warm-up: imports, caches
        for _ in range(max(args.warmup, 1) - 1):
            pool.map(_ref_task, [thetas[k] for k in range(cores)], chunksize=1)
        tot, secs, nxt = 0, 0.0, 0
        for _ in range(args.steps):
            batch = [thetas[(nxt + k) % args.ensemble] for k in range(cores)]
            nxt += cores
            t0 = time.perf_counter()
            tot += sum(pool.map(_ref_task, batch, chunksize=1))
            secs += time.perf_counter() - t0
    value = tot / secs
    sample = (f"per step: {cores} of the C5 ensemble's trajectories (consecutive starts of the seed-1 stream) x "
              f"{REF_ITERS} oracle KCM iterations, one per process of a {cores}-process pool (system and field "
              f"built once per worker); {args.steps} steps")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic", "config": config_of(args, world=int(os.environ.get("WORLD_SIZE", "1"))),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                             "host": hc, "per_core": value / cores},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# CPU legs (rank 0, N = 1): the oracle fold, one process, bounded time
# --------------------------------------------------------------------------

def cpu_fold_rate(config: str, budget_s: float, min_iters: int = 1, fixed_iters: int | None = None):
    """(it/s, iterations timed) of the oracle fold of one `config` trajectory.
    The first iteration is a warm-up unless `fixed_iters` is given (then all of
    them are timed, as for C1's 1000-iteration run)."""
    from oracle import kcm_oracle as O
    from paper_1712_05012_b200 import workloads
    try:   # one thread, as reported (cores: 1)
        from threadpoolctl import threadpool_limits
        limit = threadpool_limits(1)
    except ImportError:
        limit = None
    ch, params, w, fld = workloads.system(config)
    of = O.OracleField(params, w, solvation=fld.config.solvation)
    theta = workloads.start_theta(config, ch)
    frozen = np.zeros(ch.n_dof, bool)
    if fixed_iters is None:
        t0 = time.perf_counter()
        O.fold(ch, theta, frozen, of, max_iters=1, torque_tol_rel=0.0, energy_window=0)
        one = time.perf_counter() - t0
        iters = max(min_iters, int(budget_s / max(one, 1e-6)))
    else:
        iters = fixed_iters
    t0 = time.perf_counter()
    O.fold(ch, theta, frozen, of, max_iters=iters, torque_tol_rel=0.0, energy_window=0)
    rate = iters / (time.perf_counter() - t0)
    if limit is not None:
        limit.restore_original_limits()
    return rate, iters


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------

def time_graph(runner, K, s):
    """Device time (ms) of K graph-replayed iterations of a prepared runner."""
    import torch
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a0.record(s)
        runner.run_graph(K)
        a1.record(s)
    s.synchronize()
    return a0.elapsed_time(a1)


def ensemble_leg(P, DV, workloads, ch, fld, thetas, K, W, s):
    """(traj-it/s over K graph-replayed iterations, ms/step) of a full ensemble."""
    B = len(thetas)
    step = P.StepConfig(kappa=0.5, max_iters=W + K, torque_tol_rel=0.0, energy_window=0)
    r = DV.EnsembleRunner(ch, fld, B, step, chunk=8)
    r.load(thetas, np.zeros((B, ch.n_dof), bool))
    r.prepare(W)
    r.prepare(K)
    with __import__("torch").cuda.stream(s):
        r.run_graph(W)
    s.synchronize()
    ms = time_graph(r, K, s)
    if any(st.error for st in r.batch.status()):
        raise SystemExit("device error in an ensemble leg")
    return B * K / (ms * 1e-3), ms / K, r


def solv_roofline(workload: str, solv_ms: float, peak64: float, ref_dflop: float, T: float) -> dict:
    """The solvation kernel against the FP64 peak: executed DFLOP per launch from the
    committed ncu capture of the same workload (profiles/solvation_kernel_dflop.json)
    over the live launch time; the reference-equivalent work (8 DFLOP per coverage
    test) reported beside it."""
    out = {"bound": "fp64", "unit": "TFLOP/s", "peak": peak64 / 1e12, "achieved": None, "frac": None,
           "reference_equivalent_tflops": ref_dflop / (solv_ms * 1e-3) / 1e12,
           "work": f"executed DADD + DMUL + 2 DFMA (ncu) per launch; reference-equivalent: 8 DFLOP x T, T = "
                   f"{T:.4g} coverage tests per trajectory (mean over 4 start conformations, this package's "
                   "sasa_pass); the kernel's group masks, full-cover shortcut and early exits skip ~99 % of them"}
    path = os.path.join(ROOT, "profiles", "solvation_kernel_dflop.json")
    try:
        for rec in json.load(open(path)):
            if rec.get("workload") == workload:
                got = rec["executed_dflop_per_launch"] / (solv_ms * 1e-3)
                out.update(achieved=got / 1e12, frac=got / peak64, source=rec.get("source"))
    except (OSError, ValueError, KeyError):
        pass
    return out


def coverage_tests(P, ch, params, fld, thetas) -> float:
    """Reference-equivalent solvation coverage tests of one evaluation (SURVEY.md
    §8(d)): T = sum_i N |A_i| + sum_{gamma_i != 0} 3 (|K0_i| |A_i| + |K1_i|), with A_i
    the 8 A cavity lists and K0 / K1 the exposed / singly covered samples, from
    this package's own sasa_pass on the given start conformations (mean)."""
    sphere = fld.sphere()
    cfg = fld.config.solvation_cfg
    gamma = np.asarray(params.gamma, float) != 0.0
    out = []
    for th in thetas:
        pos = P.forward_kinematics(ch, P.Conformation(th, np.zeros(ch.n_dof, bool), ch.n_residues))
        lists = P.filtered_lists(P.build_neighbor_table(P.build_grid(pos), fld.config.cutoffs.cav), pos,
                                 fld.config.cutoffs.cav)
        _, states = P.sasa_pass(pos, params, lists, sphere, cfg)
        a = np.array([len(x) for x in lists], float)
        k0 = (states.counts == 0).sum(axis=1)
        k1 = (states.counts == 1).sum(axis=1)
        out.append(float((sphere.n * a).sum() + (3.0 * (k0 * a + k1))[gamma].sum()))
    return float(np.mean(out))


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank)

    import torch
    import torch.distributed as dist

    import paper_1712_05012_b200 as P
    from paper_1712_05012_b200 import _native as N
    from paper_1712_05012_b200 import device as DV
    from paper_1712_05012_b200 import ensemble as ENS
    from paper_1712_05012_b200 import workloads

    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    ch, params, w, fld = workloads.system("C2", solvation=args.water)
    total = args.ensemble if args.strong else args.ensemble * world
    thetas_all = workloads.random_thetas(ch, total, seed=1)
    lo, hi = ENS.shard(total, rank, world)
    B = hi - lo
    K, W, PROF = args.steps, max(args.warmup, 3), 3
    step = P.StepConfig(kappa=0.5, max_iters=W + K + PROF, torque_tol_rel=0.0, energy_window=0)
    runner = DV.EnsembleRunner(ch, fld, B, step, chunk=8)
    s = DV.stream()
    D = ch.n_dof
    theta_dev = torch.as_tensor(thetas_all[lo:hi], device=dev)
    runner.load_device(theta_dev)
    runner.batch.t["frozen"].zero_()
    runner.prepare(W)
    runner.prepare(K)
    with torch.cuda.stream(s):
        runner.run_graph(W)
    s.synchronize()

    # ---- timed region: K iterations of every trajectory + the end-of-run gather
    clocks = Clocks(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        runner.run_graph(K)
        rec = {"theta": runner.batch.t["theta"][:, :D],
               "last": runner.batch.t["rec_energy"][:, W + K - 1]}
        if world > 1:
            for key, t in rec.items():
                ENS.gather_rows(t.contiguous(), total, rank, world)
        e1.record(s)
    s.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    ms_t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = total * K / (ms_max * 1e-3)
    sts = runner.batch.status()
    if any(st.error for st in sts):
        raise SystemExit(f"device error in the ensemble: {[st.error for st in sts if st.error][:4]}")

    # ---- profile pass: per-phase CUDA events on the launching stream (eager)
    lib = N.lib()
    cs, fs, bs = N.ref(runner.dc.struct), N.ref(runner.df.struct_for(False)), N.ref(runner.batch.struct)
    ss = N.ref(DV._step_struct(step))
    names = ["fk", "bin", "pairs", "solvation", "torque"]
    acc = {k: 0.0 for k in names}
    launches_per_iter = 0
    with torch.cuda.stream(s):
        for _ in range(PROF):
            c0 = lib.kf_launch_counter()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            ev[0].record(s)
            N.check(lib.kf_fk(cs, bs, DV._sp()), "fk")
            ev[1].record(s)
            N.check(lib.kf_bin(fs, bs, DV._sp()), "bin")
            ev[2].record(s)
            N.check(lib.kf_pairs(fs, bs, DV._sp()), "pairs")
            ev[3].record(s)
            if args.water:
                N.check(lib.kf_solvation(fs, bs, DV._sp()), "solv")
            ev[4].record(s)
            N.check(lib.kf_torques_step(cs, fs, bs, ss, DV._sp()), "torque")
            ev[5].record(s)
            launches_per_iter = int(lib.kf_launch_counter() - c0)   # the graph iteration's kernels
            s.synchronize()
            for k, nm in enumerate(names):
                acc[nm] += ev[k].elapsed_time(ev[k + 1]) / PROF
    sts = runner.batch.status()
    p9 = sum(st.n_pairs for st in sts)
    p5 = sum(st.n_pairs_vdw for st in sts)
    p9_t = torch.tensor([float(p9)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(p9_t)
    pairs_per_step = float(p9_t.item())
    import ctypes as C
    out = C.c_double(0.0)
    N.check(lib.kf_peak_flops(0, C.byref(out), DV._sp()), "peak32")
    peak32 = out.value
    N.check(lib.kf_peak_flops(1, C.byref(out), DV._sp()), "peak64")
    peak64 = out.value
    flops = 25.0 * p9 + 17.0 * p5
    pair_ms = acc["pairs"]
    achieved = flops / (pair_ms * 1e-3) / 1e12
    step_ms_eager = sum(acc.values())
    launches = launches_per_iter * K

    # ---- e2e: the public API with host conformations in, host results out
    confs = [P.Conformation(thetas_all[r], np.zeros(D, bool), ch.n_residues) for r in range(lo, hi)]
    e2e_step = P.StepConfig(kappa=0.5, max_iters=K, torque_tol_rel=0.0, energy_window=0)

    def e2e_rate(f_):
        P.fold_ensemble(ch, confs, f_, e2e_step)      # warm: buffers and graphs cached
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = P.fold_ensemble(ch, confs, f_, e2e_step)
        if world > 1:
            ENS.gather_records(ENS.pack_result(res), total, device=dev)
        torch.cuda.synchronize()
        t = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return total * K / float(t.item())

    e2e_value = e2e_rate(fld)
    h2d = total * D * (8 + 1) / K
    d2h = total * (D * 8 + K * 4 * 8 + 64) / K

    extras, water, fp64, cpu, cpu_configs = {}, None, None, None, {}
    if rank == 0 and world == 1 and not args.no_extras:
        Ke = max(3, min(K, 10))
        # C5 in water (the reference's dominant CPU cost: solvation.py:135-255)
        if not args.water:
            wch, wparams, ww, wfld = workloads.system("C2", solvation=True)
            w_rate, w_ms, wr = ensemble_leg(P, DV, workloads, wch, wfld, thetas_all, Ke, 3, s)
            wcs, wfs, wbs = N.ref(wr.dc.struct), N.ref(wr.df.struct_for(False)), N.ref(wr.batch.struct)
            wr.load(thetas_all, np.zeros((args.ensemble, D), bool))   # fresh status: every trajectory live
            with torch.cuda.stream(s):
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                N.check(lib.kf_fk(wcs, wbs, DV._sp()), "fk")
                N.check(lib.kf_bin(wfs, wbs, DV._sp()), "bin")
                N.check(lib.kf_pairs(wfs, wbs, DV._sp()), "pairs")
                a0.record(s)
                N.check(lib.kf_solvation(wfs, wbs, DV._sp()), "solv")
                a1.record(s)
            s.synchronize()
            solv_ms = a0.elapsed_time(a1)
            T = coverage_tests(P, wch, wparams, wfld, thetas_all[:4])
            tests_per_launch = T * args.ensemble
            dflop = 8.0 * tests_per_launch
            confs_w = [P.Conformation(thetas_all[r], np.zeros(D, bool), ch.n_residues) for r in range(lo, hi)]
            ws = P.StepConfig(kappa=0.5, max_iters=Ke, torque_tol_rel=0.0, energy_window=0)
            P.fold_ensemble(wch, confs_w, wfld, ws)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            P.fold_ensemble(wch, confs_w, wfld, ws)
            torch.cuda.synchronize()
            w_e2e = args.ensemble * Ke / (time.perf_counter() - t0)
            water = {"workload": workload_name(args, water=True), "value": w_rate, "unit": UNIT,
                     "ms_per_step": w_ms, "steps": Ke,
                     "e2e": {"value": w_e2e, "unit": UNIT, "h2d_bytes_per_step": args.ensemble * D * 9 / Ke,
                             "d2h_bytes_per_step": args.ensemble * (D * 8 + Ke * 32 + 64) / Ke},
                     "solvation_ms_per_step": solv_ms,
                     "coverage_tests_per_s": tests_per_launch / (solv_ms * 1e-3),
                     "solvation_roofline": solv_roofline(workload_name(args, water=True), solv_ms, peak64, dflop, T)}
            del wr
        # C5 with fp64 pair math (the strict trajectory-parity mode)
        P.set_pair_precision("fp64")
        try:
            f64fld = P.Field(params, w, P.FieldConfig(solvation=args.water))
            f_rate, f_ms, fr = ensemble_leg(P, DV, workloads, ch, f64fld, thetas_all, Ke, 3, s)
            fp64 = {"value": f_rate, "unit": UNIT, "ms_per_step": f_ms, "steps": Ke,
                    "kernel": "pair_kernel<1,0> (compacted list, fp64 pair math)"}
            del fr
        finally:
            P.set_pair_precision("fp32")
        # single trajectories on one GPU (graph-replayed), C1 over the 1000-iteration config
        for cfg in ("C1", "C2", "C3", "C4"):
            c_ch, c_p, c_w, c_f = workloads.system(cfg, solvation=args.water)
            Kc = 1000 if cfg == "C1" else K
            r1 = DV.EnsembleRunner(c_ch, c_f, 1, P.StepConfig(max_iters=W + Kc, torque_tol_rel=0.0,
                                                            energy_window=0), chunk=16)
            r1.load(workloads.start_theta(cfg, c_ch)[None, :], np.zeros((1, c_ch.n_dof), bool))
            r1.prepare(W)
            r1.prepare(Kc)
            with torch.cuda.stream(s):
                r1.run_graph(W)
            s.synchronize()
            msc = time_graph(r1, Kc, s)
            st1 = r1.batch.status()[0]
            extras[cfg] = {"atoms": c_ch.n_atoms, "it_per_s": Kc / (msc * 1e-3), "iterations": Kc,
                           "pairs_9A": int(st1.n_pairs)}
        # C3 through the public fold() API (host Trajectory records out, wall clock)
        c_ch, c_p, c_w, c_f = workloads.system("C3", solvation=args.water)
        conf3 = P.Conformation(workloads.start_theta("C3", c_ch), np.zeros(c_ch.n_dof, bool), c_ch.n_residues)
        st3 = P.StepConfig(kappa=0.5, max_iters=K, torque_tol_rel=0.0, energy_window=0)
        P.fold(c_ch, conf3, c_f, st3)
        t0 = time.perf_counter()
        tr3 = P.fold(c_ch, conf3, c_f, st3)
        extras["C3"]["fold_api_it_per_s"] = tr3.iterations / (time.perf_counter() - t0)
        # CPU reference path (oracle port), one process
        cpu_rate, cpu_iters = cpu_fold_rate("C2", args.cpu_seconds, min_iters=2)
        c1_rate, c1_iters = cpu_fold_rate("C1", 0.0, fixed_iters=1000)
        c3_rate, c3_iters = cpu_fold_rate("C3", args.cpu_seconds / 3, min_iters=2)
        c4_rate, c4_iters = cpu_fold_rate("C4", 0.0, fixed_iters=1)
        cpu_configs = {"C1": {"it_per_s": c1_rate, "iterations_timed": c1_iters,
                              "note": "BASELINE config 1: 30 x ALA, 1000 KCM iterations, reference CPU path"},
                       "C2": {"it_per_s": cpu_rate, "iterations_timed": cpu_iters},
                       "C3": {"it_per_s": c3_rate, "iterations_timed": c3_iters},
                       "C4": {"it_per_s": c4_rate, "iterations_timed": c4_iters,
                              "note": "one timed iteration (the reference's ~20 s per iteration)"}}
        for cfg, v in cpu_configs.items():
            extras[cfg]["cpu_it_per_s"] = v["it_per_s"]
            extras[cfg]["speedup_vs_cpu"] = extras[cfg]["it_per_s"] / v["it_per_s"]
        hc = host_cores()
        cpu = {"value": cpu_rate, "unit": UNIT, "cores": 1, "kind": "port", "host": hc,
               "sample": f"oracle fold of one C2 trajectory, {cpu_iters} iterations, 1 thread (value in "
                         f"trajectory-iterations/s; the C5 ensemble is {args.ensemble} such trajectories, so "
                         f"the 1-core ensemble rate equals this)",
               "configs": cpu_configs}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm_peak = json.load(open(peaks_path)).get("hbm_gbs") if os.path.exists(peaks_path) else None
    # HBM rooflines of the byte-bound phases (north star: binning, scans, kinematics):
    # algorithmic bytes per trajectory (SURVEY.md §8(d) formulas) x B / phase time
    n_at, L = ch.n_atoms, len(ch.links)
    phase_bytes = {
        # theta in; link transforms (16 f64: the eager API launch writes whole rows; the fold
        # loop writes only the joint point / axis half) and positions out
        "fk": 8 * D + 128 * L + 24 * n_at,
        # joint points / axes, positions, forces, per-atom energies/counts in; tau, theta out
        "torque": 64 * L + 48 * n_at + 24 * n_at + 16 * D,
    }
    if acc.get("bin", 0.0) > 0.01:   # binning runs only where a cell table is needed (water)
        H = 1 << max(6, int(np.ceil(np.log2(n_at + 1))))
        phase_bytes["bin"] = 24 * n_at + H * (8 + 16 + 32) + n_at * (5 * 16 + 32 + 12)
    phase_roofline = {}
    for ph, by in phase_bytes.items():
        t = acc.get(ph, 0.0)
        if t > 0 and hbm_peak:
            gbs = by * B / (t * 1e-3) / 1e9
            phase_roofline[ph] = {"bound": "hbm", "bytes_per_launch": by * B, "achieved": gbs, "peak": hbm_peak,
                                  "unit": "GB/s", "frac": gbs / hbm_peak}
    # the dominant kernel of this run and its DRAM traffic / issue counts per launch from
    # the committed `ncu --set full` capture of the same workload, if there is one
    kind = int(lib.kf_pair_kernel_kind(fs, bs, n_at))
    kernel = ["pair_kernel<1,0>", "pair_dense_kernel<0,1,0>", "pair_dense_kernel<0,0,1>",
              "cluster_pair_kernel"][kind]
    traffic, traffic_src, prof = None, None, {}
    prof_path = os.path.join(ROOT, "profiles", "pair_kernel_traffic.json")
    if os.path.exists(prof_path):
        try:
            for rec in json.load(open(prof_path)):
                if rec.get("kernel") == kernel and rec.get("workload") == workload_name(args) \
                        and rec.get("ensemble") == B:
                    traffic, traffic_src, prof = rec.get("bytes_per_launch"), rec.get("source"), rec
        except (OSError, ValueError, AttributeError):
            traffic = None
    mhz = (clk or {}).get("sm_mhz") or 1965.0
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    # instruction issue (the kernel's actual bound): the capture's warp-instructions per
    # launch over the live launch time, against 4 schedulers x 1 warp-instruction/clk per SM
    issue = None
    wi = prof.get("warp_instructions_per_launch")
    if wi and pair_ms > 0:
        ipk = 4.0 * sm_count * mhz * 1e6 / 1e9
        got = wi / (pair_ms * 1e-3) / 1e9
        issue = {"achieved": got, "peak": ipk, "unit": "G warp-instructions/s", "frac": got / ipk,
                 "warp_instructions_per_launch": wi, "per_pair": wi / max(1.0, float(p9)),
                 "fma_pipe_pct_of_active": prof.get("fma_pipe_pct"),
                 "issue_active_pct": prof.get("issue_active_pct"),
                 "peak_source": f"4 issue slots/clk/SM x {sm_count} SMs at {mhz:.0f} MHz"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None,
        "dtype": "f64+f32", "data": "synthetic", "config": config_of(args, n_at, D, world),
        "pair_interactions_per_s": pairs_per_step * K / (ms_max * 1e-3),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "paper_1712_05012_b200.fold_ensemble (host numpy in, host Trajectory data out)"},
        "roofline": {"kernel": kernel + " (K3)", "bound": "fp32", "achieved": achieved,
                     "peak": peak32 / 1e12, "unit": "TFLOP/s", "frac": achieved / (peak32 / 1e12),
                     "traffic": traffic, "traffic_source": traffic_src,
                     "work": f"25*P9 + 17*P5 FLOP per trajectory (SURVEY.md §8(d)); P9={p9}, P5={p5} "
                             f"on this rank's {B} trajectories",
                     "peak_source": "kf_peak_flops FFMA microbenchmark, this GPU, this run",
                     "fp64_peak_tflops": peak64 / 1e12,
                     "kernel_share_of_step": pair_ms / step_ms_eager, "issue": issue},
        "phase_ms_per_step": acc,
        "phase_rooflines": phase_roofline,
        "gpu_launches": launches,
        "clocks": clk,
        "cpu_baseline": cpu,
        "water": water,
        "fp64_pairs": fp64,
        "single_trajectory": extras or None,
        "hbm_peak_gbs": hbm_peak,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
