"""GPU parity of exactly what the bench times, against the reference's own numbers.

The goldens (tests/golden/make_golden_bench.py) are outputs of the real
``kinefold`` on the bench's inputs:

* the first 32 trajectories of the C5 ensemble (``--init random --seed 1``),
  one KCM iteration each;
* the C3 (14,954 atoms) and C4 (99,990 atoms) single-trajectory starts;
* the C2 start in water.

Each ensemble test runs ``fold_ensemble``'s runner at the batch size that
selects a given kernel decomposition.  The kernel choice (kf_pairs_launch,
kf_bin_launch, kf_torque_launch) depends on the batch B:

* B = 1024 is the bench's C5 configuration (cluster-pair kernel, four graph
  branches of 256);
* B = 384 runs as four branches of 96 (256-thread torque CTAs from 64 trajectories);
* B = 128, 32, 30 and 16 split each trajectory over a cluster of 2 (as two
  64-trajectory branches: 4), 8, 8 and 16 CTAs.
The dense-lane kernels are covered by the C3 / C4 single-chain tests below.

The comparison covers the first min(B, 32) trajectories, against the goldens.  The
iteration's forces are read from the batch's force buffer (the test hook).

Bars:

* per-atom |dF| <= 1e-5 sum_j |f_aj|, with the reference's own scale;
* energies <= 1e-6 of (|g_elec| + |g_vdw| + |g_cav|);
* tau_max <= 1e-5 relative;
* theta' within 1e-5 kappa;
* the pair counts P9 and P5 bit-exact, since membership is decided exactly.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import kcm_oracle as O

pytestmark = pytest.mark.gpu

KAPPA = 0.5
_cache = {}


def _P():
    import paper_1712_05012_b200 as P
    return P


def _system(config, solvation=False):
    key = (config, solvation)
    if key not in _cache:
        from paper_1712_05012_b200 import workloads
        _cache[key] = workloads.system(config, solvation=solvation)
    return _cache[key]


def _wrapped(a, b):
    return np.abs((np.asarray(a) - np.asarray(b) + 180.0) % 360.0 - 180.0)


def _check_forces(forces, g_forces, g_scale, what):
    err = np.linalg.norm(forces - g_forces.astype(np.float64), axis=-1)
    scale = np.maximum(g_scale.astype(np.float64), 1e-300)
    ratio = err / scale
    assert np.all(ratio <= 1e-5), (what, float(ratio.max()), np.unravel_index(ratio.argmax(), ratio.shape))
    return float(ratio.max())


def _one_iteration_ensemble(B, solvation=False, iters=1):
    from paper_1712_05012_b200 import device as DV
    from paper_1712_05012_b200 import workloads
    P = _P()
    ch, params, w, fld = _system("C2", solvation)
    thetas = workloads.random_thetas(ch, B, seed=1)
    step = P.StepConfig(kappa=KAPPA, max_iters=iters, torque_tol_rel=0.0, energy_window=0)
    runner = DV.EnsembleRunner(ch, fld, B, step)
    runner.load(thetas, np.zeros((B, ch.n_dof), bool))
    runner.run()
    forces = runner.batch.t["forces"][:32].cpu().numpy()   # hook: this iteration's forces
    sa = runner.batch.status_array()
    return thetas, forces, runner.result(), sa


@pytest.mark.parametrize("B", [16, 30, 32, 128, 384, 1024])
def test_ensemble_iteration_matches_reference(B):
    """One iteration of the bench ensemble: forces, energies, tau_max, theta'
    and pair counts of the first min(B, 32) trajectories vs kinefold."""
    g = {k: v[:B] for k, v in golden("bench_c2_batch32").items()}
    k = min(B, 32)
    thetas, forces, res, sa = _one_iteration_ensemble(B)
    assert np.array_equal(thetas[:k], g["theta0"])
    _check_forces(forces, g["forces"], g["scale"], f"B={B}")
    E = res.energies[:k, 0, :3]
    scale = np.abs(g["energies"]).sum(axis=1)
    assert np.all(np.abs(E - g["energies"]).sum(axis=1) <= 1e-6 * scale)
    tm = res.energies[:k, 0, 3]
    assert np.all(np.abs(tm - g["tau_max"]) <= 1e-5 * g["tau_max"])
    assert _wrapped(res.theta[:k], g["theta_next"]).max() <= 1e-5 * KAPPA
    assert np.array_equal(sa["n_pairs"][:k], g["p9"])
    assert np.array_equal(sa["n_pairs_vdw"][:k], g["p5"])
    assert res.iterations.tolist() == [1] * B


def test_ensemble_rows_independent_of_batch_position():
    """The 32 pinned starts placed at the end of a 1024 batch give the same
    results as at its start: no cross-trajectory leakage in the batched kernels."""
    from paper_1712_05012_b200 import device as DV
    from paper_1712_05012_b200 import workloads
    P = _P()
    g = golden("bench_c2_batch32")
    ch, params, w, fld = _system("C2")
    thetas = workloads.random_thetas(ch, 1024, seed=1)
    thetas = np.concatenate([thetas[32:], thetas[:32]])
    step = P.StepConfig(kappa=KAPPA, max_iters=1, torque_tol_rel=0.0, energy_window=0)
    runner = DV.EnsembleRunner(ch, fld, 1024, step)
    runner.load(thetas, np.zeros((1024, ch.n_dof), bool))
    runner.run()
    forces = runner.batch.t["forces"][-32:].cpu().numpy()
    _check_forces(forces, g["forces"], g["scale"], "tail rows")
    sa = runner.batch.status_array()
    assert np.array_equal(sa["n_pairs"][-32:], g["p9"])


@pytest.mark.parametrize("config", ["C3", "C4"])
def test_single_evaluate_matches_reference(config):
    """Field.evaluate at the C3 / C4 start (the single-trajectory fp32 paths:
    C3 full list, C4 half list with fixed-point j forces) vs kinefold."""
    g = golden(f"bench_{config.lower()}_eval")
    ch, params, w, fld = _system(config)
    pos = O.fk(ch, g["theta0"])[3]
    res = fld.evaluate(pos)
    _check_forces(res.forces, g["forces"], g["scale"], config)
    e = np.array([res.energy.g_elec, res.energy.g_vdw, res.energy.g_cav])
    assert np.abs(e - g["energies"]).sum() <= 1e-6 * np.abs(g["energies"]).sum()


@pytest.mark.parametrize("config", ["C3", "C4"])
def test_single_fold_iteration_matches_reference(config):
    """One fold() iteration through the graph-replayed single-trajectory loop
    (multi-CTA FK and torque passes at C3 / C4): record energy, tau_max, theta'."""
    P = _P()
    g = golden(f"bench_{config.lower()}_eval")
    ch, params, w, fld = _system(config)
    conf = P.Conformation(g["theta0"], np.zeros(ch.n_dof, bool), ch.n_residues)
    tr = P.fold(ch, conf, fld, P.StepConfig(kappa=KAPPA, max_iters=1, torque_tol_rel=0.0, energy_window=0))
    r = tr.records[0]
    E = np.array([r.energy.g_elec, r.energy.g_vdw, r.energy.g_cav])
    assert np.abs(E - g["energies"]).sum() <= 1e-6 * np.abs(g["energies"]).sum()
    assert abs(r.tau_max - g["tau_max"]) <= 1e-5 * g["tau_max"]
    assert _wrapped(tr.final.theta, g["theta_next"]).max() <= 1e-5 * KAPPA


def test_water_evaluate_matches_reference():
    """C2 start in water: pair forces within the bar, solvation exact
    (f_exp bit-identical, g_cav to 1e-13)."""
    g = golden("bench_c2_water")
    ch, params, w, fld = _system("C2", solvation=True)
    pos = O.fk(ch, g["theta0"])[3]
    res = fld.evaluate(pos)
    _, _, extra = O.OracleField(params, w).evaluate(pos)
    from test_gpu_parity import pair_scale
    scale = pair_scale(params, w, pos, extra["i"], extra["j"], extra["d"])
    err = np.linalg.norm(res.forces - g["forces"], axis=1)
    assert np.all(err <= 1e-5 * np.maximum(scale, 1e-300)), float((err / scale).max())
    assert np.array_equal(res.sasa.f_exp, g["f_exp"])
    assert np.array_equal(res.sasa.a_exp, g["a_exp"])
    assert res.energy.g_cav == pytest.approx(float(g["energies"][2]), rel=1e-13)
    assert abs(res.energy.g_elec - g["energies"][0]) + abs(res.energy.g_vdw - g["energies"][1]) \
        <= 1e-6 * np.abs(g["energies"]).sum()


@pytest.mark.parametrize("B", [1, 1024])
def test_water_fold_matches_reference(B):
    """Two water iterations of the C2 start (B = 1: fold(); B = 1024: the bench's
    water ensemble, trajectory 0) vs the reference's 2-iteration fold."""
    g = golden("bench_c2_water")
    ref_E = g["fold_energies"]
    scale = np.abs(ref_E).sum(axis=1)
    if B == 1:
        P = _P()
        ch, params, w, fld = _system("C2", solvation=True)
        conf = P.Conformation(g["theta0"], np.zeros(ch.n_dof, bool), ch.n_residues)
        tr = P.fold(ch, conf, fld, P.StepConfig(kappa=KAPPA, max_iters=2, torque_tol_rel=0.0, energy_window=0))
        E = np.array([[r.energy.g_elec, r.energy.g_vdw, r.energy.g_cav] for r in tr.records])
        tm = np.array([r.tau_max for r in tr.records])
        final = tr.final.theta
    else:
        thetas, _, res, _ = _one_iteration_ensemble(B, solvation=True, iters=2)
        assert np.array_equal(thetas[0], g["theta0"])
        E, tm, final = res.energies[0, :, :3], res.energies[0, :, 3], res.theta[0]
    assert np.all(np.abs(E - ref_E).sum(axis=1) <= 1e-5 * scale)
    # the start conformation is the reference's bit for bit: its exposure is exact
    assert abs(E[0, 2] - ref_E[0, 2]) <= 1e-12 * abs(ref_E[0, 2])
    assert np.all(np.abs(tm - g["fold_tau_max"]) <= 1e-5 * g["fold_tau_max"])
    assert _wrapped(final, g["fold_final"]).max() <= 1e-5 * KAPPA


@pytest.mark.parametrize("B", [30, 256])
def test_ensemble_bitwise_repeatable(B):
    """Run-to-run bitwise determinism of the batched kernels (dense half list at
    B = 30, cluster pairs at B = 256): every force sum is an order-free integer
    fixed point or a fixed-order tree, so a data race (shared-memory or global)
    would show up here as a difference.  (compute-sanitizer is closed on this
    GPU pool: profiles/r2_compute_sanitizer_refused.txt.)"""
    from paper_1712_05012_b200 import device as DV
    from paper_1712_05012_b200 import workloads
    P = _P()
    ch, params, w, fld = _system("C2")
    thetas = workloads.random_thetas(ch, B, seed=2)
    step = P.StepConfig(kappa=0.5, max_iters=5, torque_tol_rel=0.0, energy_window=0)
    out = []
    for _ in range(2):
        runner = DV.EnsembleRunner(ch, fld, B, step)
        runner.load(thetas, np.zeros((B, ch.n_dof), bool))
        runner.run()
        res = runner.result()
        out.append((res.theta.copy(), res.energies.copy(), runner.batch.t["forces"].cpu().numpy()))
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("variant", ["constant_dielectric", "uniform_weights", "with_glycine"])
def test_cluster_kernel_variants_match_oracle(variant):
    """The cluster-pair kernel's other code paths against the oracle, one iteration
    at B = 192 (cluster path): constant dielectric (the DCONST build),
    UniformWeights (no class lookups), and a chain with glycines (other class
    windows).  Forces of 4 trajectories to the per-atom bar, energies to 1e-6."""
    from paper_1712_05012_b200 import device as DV
    from paper_1712_05012_b200 import workloads
    P = _P()
    seq = workloads.sequence("C2")
    if variant == "with_glycine":
        seq = [r if k % 3 else "GLY" for k, r in enumerate(seq)]
    ch = P.build_chain(seq)
    ps = P.load_params()
    params = ps.resolve(ch)
    w = P.TreeWeights(P.build_tree(ch), ps.weights)
    kw, okw = {}, {}
    if variant == "constant_dielectric":
        kw["dielectric"] = P.DielectricModel(mode="constant", kappa=4.0)
        okw = dict(dielectric_mode="constant", kappa=4.0)
    if variant == "uniform_weights":
        w = P.UniformWeights(0.7)
    fld = P.Field(params, w, P.FieldConfig(**kw))
    B = 192
    thetas = workloads.random_thetas(ch, B, seed=3)
    runner = DV.EnsembleRunner(ch, fld, B, P.StepConfig(kappa=KAPPA, max_iters=1, torque_tol_rel=0.0,
                                                        energy_window=0))
    from paper_1712_05012_b200 import _native as N
    assert N.lib().kf_pair_kernel_kind(N.ref(runner.df.struct_for(False)), N.ref(runner.batch.struct),
                                       ch.n_atoms) == 3
    runner.load(thetas, np.zeros((B, ch.n_dof), bool))
    runner.run()
    forces = runner.batch.t["forces"].cpu().numpy()
    res = runner.result()
    of = O.OracleField(params, w, **okw)
    from test_gpu_parity import pair_scale
    for r in (0, 57, 130, 191):
        pos = O.fk(ch, thetas[r])[3]
        f_ref, e_ref, ex = of.evaluate(pos)
        scale = pair_scale(params, w, pos, ex["i"], ex["j"], ex["d"], **({"mode": "constant", "kappa": 4.0}
                                                                        if okw else {}))
        err = np.linalg.norm(forces[r] - f_ref, axis=1)
        assert np.all(err <= 1e-5 * np.maximum(scale, 1e-300)), (r, float((err / scale).max()))
        e = res.energies[r, 0, :3]
        assert np.abs(e - np.array(e_ref)).sum() <= 1e-6 * np.abs(np.array(e_ref)).sum(), r


def test_graph_branches_equal_separate_sub_batches():
    """The fold graph of a 256-trajectory vacuum ensemble runs as four 64-trajectory
    branches (kf_api.cu graph_branches / batch_view).  Each branch must give bitwise
    what a separate 64-trajectory fold_ensemble gives (same kernel decomposition):
    final theta, every iteration's energies / tau_max and theta records, iterations
    and stop reasons, with a stop rule that ends some trajectories early."""
    from paper_1712_05012_b200 import workloads
    P = _P()
    ch, params, w, fld = _system("C2")
    thetas = workloads.random_thetas(ch, 256, seed=4)
    confs = [P.Conformation(t, np.zeros(ch.n_dof, bool), ch.n_residues) for t in thetas]
    step = P.StepConfig(kappa=KAPPA, max_iters=12, torque_tol_rel=0.3, energy_window=0)
    whole = P.fold_ensemble(ch, confs, fld, step, record_theta=True)
    for r in range(4):
        part = P.fold_ensemble(ch, confs[64 * r:64 * (r + 1)], fld, step, record_theta=True)
        sl = slice(64 * r, 64 * (r + 1))
        assert np.array_equal(whole.theta[sl], part.theta)
        K = part.energies.shape[1]   # records are cut at the batch's longest trajectory
        assert np.array_equal(whole.energies[sl, :K], part.energies)
        assert not whole.energies[sl, K:].any()
        assert np.array_equal(whole.thetas[sl, :K], part.thetas)
        assert np.array_equal(whole.iterations[sl], part.iterations)
        assert whole.reasons[sl] == part.reasons
