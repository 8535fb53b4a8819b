"""Run outputs of an ensemble fold, byte-compatible with the reference's files.

SURVEY.md §8(f)2: ``kinefold fold --batch B`` (cli.py:134-171) runs B
independent folds and writes, per run, ``log.csv`` / ``dihedrals.csv`` /
``timings.csv`` (RunLog, pdbio.py:248-295), ``snap_<it>.pdb`` snapshots and
``final.pdb`` (write_pdb, pdbio.py:111-132), then ``summary.csv`` and
``manifest.json`` (pdbio.py:302-309).  Here the B trajectories run as one
device batch (``fold_ensemble``) and the files are written from its record
buffers.  The deterministic files (logs, dihedrals, PDBs, summary) have the
reference's exact formats; ``timings.csv`` carries the batch's per-iteration
wall time, not per-run phase timings.
"""

from __future__ import annotations

import csv
import json
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .chain import Conformation
from .errors import PDBFormatError
from .forcefield import EnergyBreakdown

LOG_VERSION = "kinefold run log v1"
LOG_COLUMNS = ["iteration", "g_elec", "g_vdw", "g_cav", "g_total", "tau_max"]
TIMING_PHASES = ["fk", "hash", "force", "solvation", "torque"]


def _fmt(x: float) -> str:
    """Ten significant digits, the reference's log number format (pdbio.py:298)."""
    return format(float(x), ".10g")


def _csv(path: Path, rows) -> None:
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        for row in rows:
            writer.writerow(row)


def write_pdb(chain, positions, path) -> None:
    """Fixed-column PDB export of a chain's atoms (pdbio.py:111-132 layout)."""
    xyz = np.asarray(positions, float)
    n = chain.n_atoms
    if n == 0:
        raise PDBFormatError("refusing to write a structure with no atoms")
    if xyz.shape != (n, 3):
        raise PDBFormatError("positions do not match the chain's atom count")
    out = []
    for k in range(n):
        name = chain.atom_names[k]
        name_field = name if len(name) >= 4 else " " + name.ljust(3)
        res = int(chain.atom_residue[k])
        resname = chain.residues[res] if res < chain.n_residues else "LIG"
        record = "HETATM" if chain.hetero_mask[k] else "ATOM  "
        x, y, z = xyz[k]
        out.append("".join([
            record, f"{k + 1:5d}", " ", name_field, " ", f"{resname:>3s}", " A", f"{res + 1:4d}",
            "    ", f"{x:8.3f}{y:8.3f}{z:8.3f}", f"{1.0:6.2f}{0.0:6.2f}", " " * 10,
            f"{chain.atom_elements[k]:>2s}"]))
    out.append("END")
    Path(path).write_text("\n".join(out) + "\n")


@dataclass
class RunLog:
    """Per-run CSV logs and snapshot bookkeeping (pdbio.py:252-295 formats)."""

    out_dir: Path
    snapshot_paths: list = field(default_factory=list)

    def __post_init__(self):
        self.out_dir = Path(self.out_dir)
        self.out_dir.mkdir(parents=True, exist_ok=True)

    def write_trajectory(self, chain, trajectory) -> None:
        head = [f"# {LOG_VERSION}"]
        recs = trajectory.records
        _csv(self.out_dir / "log.csv",
             [head, LOG_COLUMNS] +
             [[r.index, _fmt(r.energy.g_elec), _fmt(r.energy.g_vdw), _fmt(r.energy.g_cav),
               _fmt(r.energy.g_total), _fmt(r.tau_max)] for r in recs])
        _csv(self.out_dir / "dihedrals.csv",
             [head, ["iteration"] + [f"theta_{k}" for k in range(chain.n_dof)]] +
             [[r.index] + [_fmt(v) for v in r.theta] for r in recs])
        _csv(self.out_dir / "timings.csv",
             [head, ["iteration"] + [f"t_{p}" for p in TIMING_PHASES]] +
             [[r.index] + [f"{r.timings.get(p, 0.0):.6f}" for p in TIMING_PHASES] for r in recs])

    def snapshot(self, chain, positions, tag) -> Path:
        path = self.out_dir / f"snap_{tag}.pdb"
        write_pdb(chain, positions, path)
        self.snapshot_paths.append(str(path))
        return path


def _plain(obj):
    if isinstance(obj, np.ndarray):
        return obj.tolist()
    if isinstance(obj, (np.integer, np.floating)):
        return obj.item()
    if hasattr(obj, "__dict__"):
        return {k: v for k, v in vars(obj).items() if not k.startswith("_")}
    return str(obj)


def write_manifest(out_dir, payload: dict) -> Path:
    """manifest.json: every effective parameter of a run (pdbio.py:302-309)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    path = out / "manifest.json"
    path.write_text(json.dumps(payload, indent=2, sort_keys=True, default=_plain))
    return path


def trajectories(result, confs, step, wall_per_iteration: float = 0.0) -> list:
    """Per-run ``Trajectory`` objects from an ``EnsembleResult`` recorded with
    ``record_theta=True`` (records, snapshots every ``step.snapshot_every``,
    final conformation, stop reason: kcm.py:312-351 semantics)."""
    from .kcm import IterationRecord, Trajectory
    if result.thetas is None:
        raise ValueError("trajectories() needs fold_ensemble(..., record_theta=True)")
    out = []
    timing = {p: 0.0 for p in TIMING_PHASES}
    timing["force"] = wall_per_iteration
    for b, conf in enumerate(confs):
        frozen = np.asarray(conf.frozen, bool)
        k_end = int(result.iterations[b])
        records, snaps = [], []
        for k in range(k_end):
            e = result.energies[b, k]
            theta = np.array(result.thetas[b, k], float)
            records.append(IterationRecord(k, EnergyBreakdown(float(e[0]), float(e[1]), float(e[2])),
                                           float(e[3]), dict(timing), theta))
            if step.snapshot_every and k % step.snapshot_every == 0:
                snaps.append((k, Conformation(theta.copy(), frozen, conf.residue_count)))
        final = Conformation(np.array(result.theta[b], float), frozen, conf.residue_count)
        reason = result.reasons[b]
        out.append(Trajectory(records, snaps, final, reason != "max_iters", reason))
    return out


def fold_batch(chain, confs, fld, step, out, *, manifest: dict | None = None, verbose: bool = False) -> list:
    """``kinefold fold --batch B`` (cli.py:134-171) with the B folds as one
    device batch.  Writes ``out/run_XXXX/`` (or ``out/`` for one run) and, for
    B > 1, ``out/summary.csv``; ``manifest`` (if given) goes to
    ``out/manifest.json``.  Returns the per-run trajectories."""
    import time

    from .chain import forward_kinematics
    from .kcm import fold_ensemble
    confs = list(confs)
    out = Path(out)
    t0 = time.perf_counter()
    result = fold_ensemble(chain, confs, fld, step, record_theta=True)
    wall = (time.perf_counter() - t0) / max(1, int(np.max(result.iterations)) if len(confs) else 1)
    trajs = trajectories(result, confs, step, wall)
    rows = []
    for run, traj in enumerate(trajs):
        run_dir = out if len(trajs) == 1 else out / f"run_{run:04d}"
        log = RunLog(run_dir)
        log.write_trajectory(chain, traj)
        for it, snap in traj.snapshots:
            log.snapshot(chain, forward_kinematics(chain, snap), f"{it:06d}")
        write_pdb(chain, forward_kinematics(chain, traj.final), run_dir / "final.pdb")
        phi, psi, _ = chain.dihedrals_from_theta(traj.final)
        g_last = traj.records[-1].energy.g_total
        rows.append([run, traj.iterations, traj.converged, traj.reason, f"{g_last:.6g}",
                     f"{np.mean(phi[1:]):.2f}", f"{np.mean(psi[:-1]):.2f}"])
        if verbose:
            print(f"run {run}: {traj.iterations} iterations, converged={traj.converged} ({traj.reason}), "
                  f"G_total={g_last:.3f} kcal/mol")
    if len(trajs) > 1:
        _csv(out / "summary.csv",
             [["run", "iterations", "converged", "reason", "g_total", "mean_phi", "mean_psi"]] + rows)
    if manifest is not None:
        write_manifest(out, manifest)
    return trajs


BENCH_COLUMNS = ["m", "atoms", "t_hash_build", "t_force_hashed", "t_force_brute", "t_solvation"]


def bench_table(sizes, out, *, water: bool = False, samples: int = 1024, repeat: int = 3,
                gamma_set: str = "sharp", params_path=None, verbose: bool = False) -> list:
    """``kinefold bench`` (cli.py:245-286): poly-ALA chains of ``sizes``
    residues at the zero-point conformation, one ``Field.evaluate`` with the
    hash grid and one with ``use_hash=False`` (the quadratic path) per repeat,
    best-of-``repeat`` phase times (device-event seconds here).  Writes
    ``out/bench.csv`` (the reference's columns and 6-decimal format) and
    ``out/manifest.json``; returns the rows."""
    import dataclasses

    from . import __version__
    from .chain import build_chain, forward_kinematics
    from .kcm import Field, FieldConfig
    from .params import load_params
    from .solvation import SolvationConfig
    from .topology import TreeWeights, build_tree
    out = Path(out)
    out.mkdir(parents=True, exist_ok=True)
    ps = load_params(params_path)
    rows = []
    for m in [int(s) for s in sizes]:
        chain = build_chain(["ALA"] * m)
        weights = TreeWeights(build_tree(chain), ps.weights)
        base = FieldConfig(solvation=bool(water), solvation_cfg=SolvationConfig(samples=samples))
        params = ps.resolve(chain, gamma_set)
        fld_h = Field(params, weights, base)
        fld_b = Field(params, weights, dataclasses.replace(base, use_hash=False))
        pos = forward_kinematics(chain, chain.conf_zp())
        t_hash = t_force_h = t_force_b = t_solv = float("inf")
        for _ in range(max(1, int(repeat))):
            r = fld_h.evaluate(pos)
            t_hash = min(t_hash, r.timings["hash"])
            t_force_h = min(t_force_h, r.timings["force"])
            t_solv = min(t_solv, r.timings["solvation"])
            rb = fld_b.evaluate(pos)
            # the quadratic mode's layout pass is force work (cli.py:272-273)
            t_force_b = min(t_force_b, rb.timings["force"] + rb.timings["hash"])
        rows.append([m, chain.n_atoms, t_hash, t_force_h, t_force_b, t_solv])
        if verbose:
            print(f"{m:6d} {chain.n_atoms:7d} {t_hash:10.5f} {t_force_h:11.5f} {t_force_b:11.5f} {t_solv:10.5f}")
    _csv(out / "bench.csv", [BENCH_COLUMNS] + [[r[0], r[1]] + [f"{x:.6f}" for x in r[2:]] for r in rows])
    write_manifest(out, {"version": __version__, "command": "bench",
                         "arguments": {"sizes": ",".join(str(s) for s in sizes), "water": bool(water),
                                       "samples": samples, "repeat": repeat, "gamma_set": gamma_set}})
    return rows
