"""Goldens for exactly what the bench times, from the REAL reference package.

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden_bench.py            # all
    python tests/golden/make_golden_bench.py c2 c3      # a subset

Every number saved is an output of ``kinefold`` 0.1.0 itself, on the inputs of
SURVEY.md §8(d) (the bench's workloads):

* ``bench_c2_batch32``: the first 32 starts of the bench's C5 ensemble
  (``kinefold fold --init random --seed 1 --batch 1024`` stream, cli.py:136,
  :146-147), one KCM iteration each: Field.evaluate (kcm.py:104-150) forces
  and energies, link_wrenches + joint_torques (kcm.py:177-240) tau, kcm_step
  (kcm.py:264-274) theta', the pair counts P9 / P5 and the per-atom
  cancellation scale sum_j |f_aj| of the force bar.
* ``bench_c3_eval`` / ``bench_c4_eval``: the same for the C3 (14,954 atoms) and
  C4 (99,990 atoms) single-trajectory starts (seed 1).
* ``bench_c2_water``: the C2 start in water (FieldConfig(solvation=True)): one
  evaluate (forces, energies, f_exp) and a 2-iteration fold.

Positions are not stored: the oracle's FK reproduces the reference's bit for
bit (tests/test_oracle_golden.py), so the tests rebuild them from theta.
Forces and scales of the large cases are stored as float32: the storage
rounding (6e-8 |F| <= 6e-8 sum_j |f_aj|) is 0.6 % of the 1e-5 bar.
"""

from __future__ import annotations

import os
import sys
from multiprocessing import get_context

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import kinefold as K  # noqa: E402
from kinefold.forcefield import (elec_pair_quantities, extract_pairs,  # noqa: E402
                                 vdw_pair_quantities)

OUT = os.path.dirname(os.path.abspath(__file__))
RESIDUES = {"C2": 140, "C3": 1400, "C4": 9375}


def system(config, solvation=False):
    seq = [str(x) for x in np.random.default_rng(0).choice(["ALA", "CYS", "SER"], RESIDUES[config])]
    ch = K.build_chain(seq)
    ps = K.load_params()
    params = ps.resolve(ch)
    w = K.TreeWeights(K.build_tree(ch), ps.weights)
    return ch, params, w, K.Field(params, w, K.FieldConfig(solvation=solvation))


def starts(ch, count, seed=1):
    """The `--init random --seed S --batch count` conformations (cli.py:116-120, :146-147)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        phi = rng.uniform(-90.0, 90.0, ch.n_residues)
        psi = rng.uniform(-90.0, 90.0, ch.n_residues)
        out.append(ch.conf_from_backbone(phi, psi))
    return out


def one_iteration(ch, params, w, fld, conf):
    st = K.kinematic_state(ch, conf)
    pos = st.positions
    res = fld.evaluate(pos)
    wr = K.link_wrenches(ch, pos, res.forces)
    tau = K.joint_torques(ch, conf, wr, st).tau
    nxt, deltas = K.kcm_step(K.JointTorques(tau), conf, K.StepConfig(kappa=0.5))
    # the force bar's per-atom scale sum_j |f_aj| and the pair counts, from the
    # reference's own pair set, weights and pair quantities (kcm.py:110-127)
    table, _ = fld._neighbor_table(pos)
    i, j, d = extract_pairs(pos, table, 9.0)
    n = len(pos)
    scale = np.zeros(n)
    ke, kv = d <= 9.0, d <= 5.0
    _, me = elec_pair_quantities(params, i[ke], j[ke], d[ke], w.weights_for(i[ke], j[ke], "elec"),
                                 fld.config.dielectric)
    _, mv = vdw_pair_quantities(params, i[kv], j[kv], d[kv], w.weights_for(i[kv], j[kv], "vdw"))
    for ii, jj, m in ((i[ke], j[ke], np.abs(me)), (i[kv], j[kv], np.abs(mv))):
        scale += np.bincount(ii, weights=m, minlength=n) + np.bincount(jj, weights=m, minlength=n)
    return dict(theta0=conf.theta, energies=np.array([res.energy.g_elec, res.energy.g_vdw, res.energy.g_cav]),
                forces=res.forces, scale=scale, tau=tau, tau_max=np.abs(tau).max(),
                theta_next=nxt.theta, p9=int(ke.sum()), p5=int(kv.sum()))


def _c2_worker(r):
    ch, params, w, fld = system("C2")
    conf = starts(ch, r + 1)[r]
    return one_iteration(ch, params, w, fld, conf)


def make_c2():
    with get_context("fork").Pool(min(8, os.cpu_count() or 1)) as pool:
        rows = pool.map(_c2_worker, range(32))
    out = {k: np.stack([r[k] for r in rows]) for k in rows[0]}
    out["forces"] = out["forces"].astype(np.float32)
    out["scale"] = out["scale"].astype(np.float32)
    np.savez_compressed(os.path.join(OUT, "bench_c2_batch32.npz"), **out)
    print("bench_c2_batch32", out["forces"].shape, out["p9"][:4])


def make_single(config):
    ch, params, w, fld = system(config)
    conf = starts(ch, 1)[0]
    out = one_iteration(ch, params, w, fld, conf)
    out["forces"] = out["forces"].astype(np.float32)
    out["scale"] = out["scale"].astype(np.float32)
    np.savez_compressed(os.path.join(OUT, f"bench_{config.lower()}_eval.npz"), **out)
    print(f"bench_{config.lower()}_eval", ch.n_atoms, out["p9"], out["energies"])


def make_water():
    ch, params, w, fld = system("C2", solvation=True)
    conf = starts(ch, 1)[0]
    pos = K.kinematic_state(ch, conf).positions
    res = fld.evaluate(pos)
    tr = K.fold(ch, conf, fld, K.StepConfig(kappa=0.5, max_iters=2, torque_tol_rel=0.0, energy_window=0))
    out = dict(theta0=conf.theta, energies=np.array([res.energy.g_elec, res.energy.g_vdw, res.energy.g_cav]),
               forces=res.forces, f_exp=res.sasa.f_exp, a_exp=res.sasa.a_exp,
               fold_energies=np.array([[r.energy.g_elec, r.energy.g_vdw, r.energy.g_cav] for r in tr.records]),
               fold_tau_max=np.array([r.tau_max for r in tr.records]), fold_final=tr.final.theta)
    np.savez_compressed(os.path.join(OUT, "bench_c2_water.npz"), **out)
    print("bench_c2_water", out["energies"], out["fold_energies"])


if __name__ == "__main__":
    want = sys.argv[1:] or ["c2", "c3", "c4", "water"]
    for key in want:
        {"c2": make_c2, "c3": lambda: make_single("C3"), "c4": lambda: make_single("C4"),
         "water": make_water}[key]()
