"""Benchmark: KCM iterations/s of the B200 KCM loop (BASELINE.json metric).

Workload: an ensemble of 1024 independent
trajectories of the 140-residue / 1,499-atom synthetic A/C/S chain (C2),
random +-90 starts (`--init random --seed 1 --batch 1024` semantics), vacuum
FieldConfig() defaults, fixed iteration count (torque_tol_rel = 0,
energy_window = 0).  A step is one KCM iteration of every trajectory (FK ->
hash binning -> elec/vdW pair forces -> wrenches -> suffix-scan torques ->
max-normalised step), replayed from CUDA graphs.  With N GPUs (torchrun) the
1024 trajectories are split into contiguous blocks, one per rank; there is no
per-iteration communication and one NCCL all-gather of the final per-trajectory
records at the end of the timed region (scaling "strong": total work fixed).

Output: one JSON line on rank 0 (see the README of the driver contract):
value = trajectory-iterations/s of the whole job; e2e = the same through the
public `fold_ensemble` API with host inputs/outputs; roofline of the dominant
kernel; cpu_baseline = the oracle (numpy restatement of the reference,
`oracle/kcm_oracle.py`) timed on this host; single-trajectory C2/C3 numbers.

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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ensemble", type=int, default=ENSEMBLE)
    ap.add_argument("--water", action="store_true", help="FieldConfig(solvation=True)")
    ap.add_argument("--no-extras", action="store_true", help="skip single-trajectory and CPU legs")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def workload_name(args) -> str:
    mode = "water" if args.water else "vacuum"
    return (f"C5: ensemble of {args.ensemble} x C2 chain (140 random A/C/S residues, 1499 atoms), "
            f"random +-90 starts, {mode}, fixed iterations")


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

def _cpu_worker(payload):
    thetas, iters = payload
    from oracle import kcm_oracle as O
    from paper_1712_05012_b200 import workloads
    ch, params, w, _ = workloads.system("C2")
    of = O.OracleField(params, w)
    for th in thetas:
        O.fold(ch, th, np.zeros(ch.n_dof, bool), of, max_iters=iters, torque_tol_rel=0.0, energy_window=0)
    return len(thetas) * iters


def reference_arm(args, rank: int):
    import multiprocessing as mp

    from paper_1712_05012_b200 import workloads
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    ch = workloads.system("C2")[0]
    thetas = workloads.random_thetas(ch, cores, seed=1)
    iters = 2
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        def one_step():
            t0 = time.perf_counter()
            done = sum(pool.map(_cpu_worker, [([thetas[k]], iters) for k in range(cores)]))
            return done, time.perf_counter() - t0
        for _ in range(max(args.warmup, 1)):
            one_step()
        tot, secs = 0, 0.0
        for _ in range(args.steps):
            d, s = one_step()
            tot, secs = tot + d, secs + s
    value = tot / secs
    sample = (f"{cores} C2 trajectories x {iters} oracle KCM iterations per step on a {cores}-process pool, "
              f"{args.steps} steps")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload_name(args), "ensemble": args.ensemble},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# CPU baseline leg (rank 0, N = 1): oracle fold, one trajectory, bounded time
# --------------------------------------------------------------------------

def cpu_fold_rate(config: str, budget_s: float, min_iters: int = 2):
    from oracle import kcm_oracle as O
    from paper_1712_05012_b200 import workloads
    ch, params, w, fld = workloads.system(config)
    of = O.OracleField(params, w, solvation=fld.config.solvation)
    theta = workloads.start_theta(config, ch)
    t0 = time.perf_counter()
    O.fold(ch, theta, np.zeros(ch.n_dof, bool), of, max_iters=1, torque_tol_rel=0.0, energy_window=0)
    one = time.perf_counter() - t0
    iters = max(min_iters, int(budget_s / max(one, 1e-6)))
    t0 = time.perf_counter()
    O.fold(ch, theta, np.zeros(ch.n_dof, bool), of, max_iters=iters, torque_tol_rel=0.0, energy_window=0)
    return iters / (time.perf_counter() - t0), iters


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------

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
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    ch, params, w, fld = workloads.system("C2", solvation=args.water)
    if args.water:
        fld = P.Field(params, w, P.FieldConfig(solvation=True))
    thetas_all = workloads.random_thetas(ch, args.ensemble, seed=1)
    lo, hi = ENS.shard(args.ensemble, rank, world)
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
                ENS.gather_rows(t.contiguous(), args.ensemble, rank, world)
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
    value = args.ensemble * K / (ms_max * 1e-3)
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
    P.fold_ensemble(ch, confs, fld, e2e_step)      # warm: buffers and graphs cached
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = P.fold_ensemble(ch, confs, fld, e2e_step)
    if world > 1:
        ENS.gather_records(ENS.pack_result(res), args.ensemble, device=dev)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    e2e_t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = args.ensemble * K / float(e2e_t.item())
    h2d = args.ensemble * D * (8 + 1) / K
    d2h = args.ensemble * (D * 8 + K * 4 * 8 + 64) / K

    extras = {}
    cpu = None
    if rank == 0 and world == 1 and not args.no_extras:
        # single-trajectory C2 / C3 on one GPU (graph-replayed), and CPU legs
        for cfg in ("C2", "C3", "C4"):   # C4: ~100k atoms (GPU only; the CPU port needs ~20 s/iteration)
            c_ch, c_p, c_w, c_f = workloads.system(cfg, solvation=args.water)
            r1 = DV.EnsembleRunner(c_ch, c_f, 1, P.StepConfig(max_iters=W + K, torque_tol_rel=0.0,
                                                            energy_window=0), chunk=16)
            r1.load(workloads.start_theta(cfg, c_ch)[None, :], np.zeros((1, c_ch.n_dof), bool))
            r1.prepare(W)
            r1.prepare(K)
            with torch.cuda.stream(s):
                r1.run_graph(W)
                s.synchronize()
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(s)
                r1.run_graph(K)
                a1.record(s)
            s.synchronize()
            st1 = r1.batch.status()[0]
            extras[cfg] = {"atoms": c_ch.n_atoms, "it_per_s": K / (a0.elapsed_time(a1) * 1e-3),
                           "pairs_9A": int(st1.n_pairs)}
        cpu_rate, cpu_iters = cpu_fold_rate("C2", args.cpu_seconds)
        extras["C2"]["cpu_it_per_s"] = cpu_rate
        extras["C2"]["speedup_vs_cpu"] = extras["C2"]["it_per_s"] / cpu_rate
        c3_rate, c3_iters = cpu_fold_rate("C3", args.cpu_seconds / 3, min_iters=2)
        extras["C3"]["cpu_it_per_s"] = c3_rate
        extras["C3"]["cpu_iters_timed"] = c3_iters
        extras["C3"]["speedup_vs_cpu"] = extras["C3"]["it_per_s"] / c3_rate
        cpu = {"value": cpu_rate, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"oracle fold of one C2 trajectory, {cpu_iters} iterations, 1 thread "
                         f"(value in trajectory-iterations/s; the C5 ensemble is {args.ensemble} such "
                         f"trajectories, so the 1-core ensemble rate equals this)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm_peak = json.load(open(peaks_path)).get("hbm_gbs") if os.path.exists(peaks_path) else None
    # HBM rooflines of the byte-bound phases (north star: binning, scans, kinematics):
    # algorithmic bytes per trajectory (SURVEY.md §8(d) formulas) x B / phase time
    n_at, L = ch.n_atoms, len(ch.links)
    H = 1 << max(6, int(np.ceil(np.log2(n_at + 1))))
    phase_bytes = {
        # theta in; link transforms (16 f64) and positions out
        "fk": 8 * D + 128 * L + 24 * n_at,
        # positions in; hash table (key 8 + count/start/occ/chunk 4x4 + box 32) and the
        # cell-ordered SoA (hi/lo/par/aux/tree 5x16 + fp64 position 32) + slot/rank/sorted out
        "bin": 24 * n_at + H * (8 + 16 + 32) + n_at * (5 * 16 + 32 + 12),
        # transforms, positions, forces, per-atom energies/counts in; tau, theta out
        "torque": 128 * L + 48 * n_at + 24 * n_at + 16 * D,
    }
    phase_roofline = {}
    for ph, by in phase_bytes.items():
        t = acc.get(ph, 0.0)
        if t > 0 and hbm_peak:
            gbs = by * B / (t * 1e-3) / 1e9
            phase_roofline[ph] = {"bound": "hbm", "bytes_per_launch": by * B, "achieved": gbs, "peak": hbm_peak,
                                  "unit": "GB/s", "frac": gbs / hbm_peak}
    # the dominant kernel of this run (kf_nonbonded.cu: half-list dense lanes for
    # fp32 ensembles, the compacted list for fp64) and its DRAM traffic per launch from
    # the committed `ncu --set full` capture of the same workload, if there is one
    kernel = "pair_kernel<1,0>" if P.pair_precision() == "fp64" else \
        ("pair_dense_kernel<0,0,1>" if B * ch.n_atoms >= 40000 else "pair_dense_kernel<0,1,0>")
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
    # shared-memory bandwidth of the pair kernel (north star): the capture's shared
    # wavefronts per launch (128 B each) over the live-measured launch time, against
    # the nominal 32 banks x 4 B per clock per SM at the clock seen under load
    smem = None
    wf = prof.get("smem_wavefronts_per_launch")
    if wf and pair_ms > 0:
        mhz = (clk or {}).get("sm_mhz") or 1965.0
        sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
        smem_peak = 128.0 * sm_count * mhz * 1e6 / 1e9
        smem_gbs = wf * 128.0 / (pair_ms * 1e-3) / 1e9
        smem = {"achieved": smem_gbs, "peak": smem_peak, "unit": "GB/s", "frac": smem_gbs / smem_peak,
                "wavefronts_per_launch": wf, "fma_pipe_pct_of_active": prof.get("fma_pipe_pct"),
                "issue_active_pct": prof.get("issue_active_pct"),
                "peak_source": f"nominal 128 B/clk/SM x {sm_count} SMs at {mhz:.0f} MHz"}
    # instruction issue (the kernel's actual bound): the capture's warp-instructions per
    # launch over the live launch time, against 4 schedulers x 1 warp-instruction/clk per SM
    issue = None
    wi = prof.get("warp_instructions_per_launch")
    if wi and pair_ms > 0:
        mhz = (clk or {}).get("sm_mhz") or 1965.0
        sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
        ipk = 4.0 * sm_count * mhz * 1e6 / 1e9
        got = wi / (pair_ms * 1e-3) / 1e9
        issue = {"achieved": got, "peak": ipk, "unit": "G warp-instructions/s", "frac": got / ipk,
                 "warp_instructions_per_launch": wi,
                 "per_pair": wi / max(1.0, float(p9)),
                 "peak_source": f"4 issue slots/clk/SM x {sm_count} SMs at {mhz:.0f} MHz"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64+f32", "data": "synthetic",
        "config": {"workload": workload_name(args), "ensemble": args.ensemble, "atoms_per_trajectory": ch.n_atoms,
                   "dofs": D, "parallelism": f"trajectory-parallel x{world}",
                   "l2": "working set per step > 126 MB L2 (sorted positions, forces, link transforms "
                         "of 1.5M atoms / 530k links), no explicit flush"},
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
                     "kernel_share_of_step": pair_ms / step_ms_eager,
                     "smem": smem, "issue": issue},
        "phase_ms_per_step": acc,
        "phase_rooflines": phase_roofline,
        "gpu_launches": launches,
        "clocks": clk,
        "cpu_baseline": cpu,
        "single_trajectory": extras or None,
        "hbm_peak_gbs": hbm_peak,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
