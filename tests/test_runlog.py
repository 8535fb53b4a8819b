"""Run outputs of `fold_batch` against files written by the
reference CLI (`kinefold fold --batch 2`, tests/golden/make_fold_batch.sh).

CPU: the writers reproduce the reference's log / dihedral files byte for byte
from the same numbers.  GPU: `fold_batch` (fp64 pair math) reproduces the
runs -- same files, headers, iteration indices, stop reasons and convergence
flags; numbers to 1e-8 relative (the printed 10 digits of fp64 trajectories
that agree to ~1e-12), PDB columns identical apart from coordinates (1e-3 A).
"""

from __future__ import annotations

import csv
import os

import numpy as np
import pytest

from conftest import ROOT

GOLD = os.path.join(ROOT, "tests", "golden", "fold_batch")
SEQ = "ALA CYS SER ALA GLY ALA SER CYS ALA ALA".split()


def _rows(path):
    with open(path, newline="") as fh:
        return list(csv.reader(fh))


def _gold_trajectory(run):
    from paper_1712_05012_b200.forcefield import EnergyBreakdown
    from paper_1712_05012_b200.kcm import IterationRecord, Trajectory
    log = _rows(os.path.join(GOLD, f"run_{run:04d}", "log.csv"))[2:]
    dih = _rows(os.path.join(GOLD, f"run_{run:04d}", "dihedrals.csv"))[2:]
    recs = [IterationRecord(int(r[0]), EnergyBreakdown(float(r[1]), float(r[2]), float(r[3])), float(r[5]), {},
                            np.array([float(x) for x in d[1:]])) for r, d in zip(log, dih)]
    return Trajectory(recs, [], None, False, "")


@pytest.mark.parametrize("run", [0, 1])
def test_runlog_writes_reference_bytes(run, tmp_path):
    import paper_1712_05012_b200 as P
    from paper_1712_05012_b200.runlog import RunLog
    ch = P.build_chain(SEQ)
    RunLog(tmp_path).write_trajectory(ch, _gold_trajectory(run))
    with open(tmp_path / "dihedrals.csv", "rb") as a, open(os.path.join(GOLD, f"run_{run:04d}", "dihedrals.csv"),
                                                           "rb") as b:
        assert a.read() == b.read()
    # log.csv: every column but g_total, which the reference sums from unrounded terms
    with open(tmp_path / "log.csv", "rb") as a, open(os.path.join(GOLD, f"run_{run:04d}", "log.csv"), "rb") as b:
        got, ref = a.read().split(b"\r\n"), b.read().split(b"\r\n")
    assert len(got) == len(ref) and got[:2] == ref[:2]
    drop = lambda line: b",".join(f for k, f in enumerate(line.split(b",")) if k != 4)  # noqa: E731
    assert [drop(x) for x in got[2:]] == [drop(x) for x in ref[2:]]


def _close_rows(got, ref, rel):
    assert len(got) == len(ref)
    for g, r in zip(got, ref):
        assert len(g) == len(r)
        for x, y in zip(g, r):
            try:
                fx, fy = float(x), float(y)
            except ValueError:
                assert x == y
                continue
            assert abs(fx - fy) <= rel * max(abs(fy), 1e-3), (x, y)


def _pdb_close(got_path, ref_path):
    got = open(got_path).read().splitlines()
    ref = open(ref_path).read().splitlines()
    assert len(got) == len(ref)
    for g, r in zip(got, ref):
        if not r.startswith(("ATOM", "HETATM")):
            assert g == r
            continue
        assert g[:30] == r[:30] and g[54:] == r[54:]
        assert np.allclose([float(g[30:38]), float(g[38:46]), float(g[46:54])],
                           [float(r[30:38]), float(r[38:46]), float(r[46:54])], atol=1.5e-3)


@pytest.mark.gpu
def test_fold_batch_matches_reference_cli(tmp_path):
    import paper_1712_05012_b200 as P
    from paper_1712_05012_b200 import workloads
    from paper_1712_05012_b200.runlog import fold_batch
    ch = P.build_chain(SEQ)
    ps = P.load_params()
    fld = P.Field(ps.resolve(ch), P.TreeWeights(P.build_tree(ch), ps.weights), P.FieldConfig())
    thetas = workloads.random_thetas(ch, 2, seed=3)          # --init random --seed 3 --batch 2
    confs = [P.Conformation(t, np.zeros(ch.n_dof, bool), ch.n_residues) for t in thetas]
    step = P.StepConfig(max_iters=25, snapshot_every=10)
    P.set_pair_precision("fp64")
    try:
        fold_batch(ch, confs, fld, step, tmp_path)
    finally:
        P.set_pair_precision("fp32")
    got_sum, ref_sum = _rows(tmp_path / "summary.csv"), _rows(os.path.join(GOLD, "summary.csv"))
    assert [r[:4] for r in got_sum] == [r[:4] for r in ref_sum]      # run, iterations, converged, reason
    _close_rows([r[4:] for r in got_sum[1:]], [r[4:] for r in ref_sum[1:]], 1e-5)
    for run in (0, 1):
        d = f"run_{run:04d}"
        for name in ("log.csv", "dihedrals.csv"):
            got, ref = _rows(tmp_path / d / name), _rows(os.path.join(GOLD, d, name))
            assert got[:2] == ref[:2]
            assert [r[0] for r in got] == [r[0] for r in ref]
            _close_rows(got[2:], ref[2:], 1e-8)
        _pdb_close(tmp_path / d / "final.pdb", os.path.join(GOLD, d, "final.pdb"))
        assert sorted(p.name for p in (tmp_path / d).glob("snap_*.pdb")) == \
            (["snap_000000.pdb", "snap_000010.pdb", "snap_000020.pdb"] if run == 0
             else ["snap_000000.pdb", "snap_000010.pdb"])
    _pdb_close(tmp_path / "run_0000" / "snap_000010.pdb", os.path.join(GOLD, "run_0000", "snap_000010.pdb"))


@pytest.mark.gpu
def test_bench_table_rows_and_trend(tmp_path):
    """``kinefold bench`` (test_cli.py:97-106): header + one row per size, and
    at the largest size the hashed force pass beats the quadratic one."""
    import json

    import paper_1712_05012_b200 as P
    out = tmp_path / "b"
    P.bench_table([20, 40, 80], out, repeat=2)
    with open(out / "bench.csv", newline="") as fh:
        rows = list(csv.reader(fh))
    assert rows[0] == ["m", "atoms", "t_hash_build", "t_force_hashed", "t_force_brute", "t_solvation"]
    assert len(rows) == 4 and [r[0] for r in rows[1:]] == ["20", "40", "80"]
    assert all(len(v.split(".")[1]) == 6 for r in rows[1:] for v in r[2:])
    assert float(rows[-1][3]) <= float(rows[-1][4])
    assert json.loads((out / "manifest.json").read_text())["command"] == "bench"
