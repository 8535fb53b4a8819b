"""GPU parity: every hot-path function through the C ABI vs the reference's
own golden vectors (tests/golden, produced by kinefold itself) and the oracle.

Bars: bit-exact for cell assignment, neighbour tables, pair
sets, exposure states, solvation forces, wrenches and the step; per-atom
|dF| <= 1e-5 * sum_j |f_aj| for the fp32 pair math; torques <= 1e-5 max|tau|;
trajectories: per-record |dE| <= 1e-5 (|g_elec| + |g_vdw| + |g_cav|).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, make_system
from oracle import kcm_oracle as O

pytestmark = pytest.mark.gpu

FORCE_TOL = 1e-5


def _P():
    import paper_1712_05012_b200 as P
    return P


def pair_scale(params, weights, pos, i, j, d, ce=9.0, cv=5.0, mode="distance", kappa=1.0):
    """Cancellation-aware per-atom scale sum_j |f_aj| (fp64, oracle formulas)."""
    n = len(pos)
    ke, kv = d <= ce, d <= cv
    _, me = O.elec_terms(params, i[ke], j[ke], d[ke], O.pair_weights(weights, i[ke], j[ke], "elec"), mode, kappa)
    _, mv = O.vdw_terms(params, i[kv], j[kv], d[kv], O.pair_weights(weights, i[kv], j[kv], "vdw"))
    s = np.zeros(n)
    for ii, jj, m in ((i[ke], j[ke], np.abs(me)), (i[kv], j[kv], np.abs(mv))):
        s += np.bincount(ii, weights=m, minlength=n) + np.bincount(jj, weights=m, minlength=n)
    return s


# ---- forward kinematics ---------------------------------------------------------

@pytest.mark.parametrize("name", ["c1_helix", "c2_random", "mixed_water"])
def test_fk_matches_reference(name):
    P = _P()
    g = golden(name)
    ch = P.build_chain(list(g["seq"]))
    conf = P.Conformation(g["theta"], np.zeros(len(g["theta"]), bool), ch.n_residues)
    st = P.kinematic_state(ch, conf)
    assert np.abs(st.positions - g["positions"]).max() < 1e-9
    assert np.abs(np.array(st.transforms) - g["link_M"]).max() < 1e-12
    assert np.abs(np.array(st.joint_points) - g["link_P"]).max() < 1e-9
    U = np.array([np.zeros(3) if u is None else u for u in st.axes])
    assert np.abs(U - g["link_U"]).max() < 1e-12
    assert np.array_equal(P.forward_kinematics(ch, conf), st.positions)


# ---- field evaluation ---------------------------------------------------------------

@pytest.mark.parametrize("name,kw", [("c1_helix", {}), ("c2_random", {}),
                                     ("mixed_const_kappa", {"const": True})])
def test_evaluate_vacuum_matches_reference(name, kw):
    P = _P()
    g = golden(name)
    diel = P.DielectricModel(mode="constant", kappa=4.0) if kw.get("const") else None
    ch, params, w, fld = make_system(g["seq"], dielectric=diel)
    res = fld.evaluate(g["positions"])
    _, _, extra = O.OracleField(params, w, dielectric_mode="constant" if diel else "distance",
                                kappa=4.0 if diel else 1.0).evaluate(g["positions"])
    scale = pair_scale(params, w, g["positions"], extra["i"], extra["j"], extra["d"],
                       mode="constant" if diel else "distance", kappa=4.0 if diel else 1.0)
    err = np.linalg.norm(res.forces - g["forces"], axis=1)
    assert np.all(err <= FORCE_TOL * np.maximum(scale, 1e-300)), (err / scale).max()
    e_ref = g["energies"]
    e = np.array([res.energy.g_elec, res.energy.g_vdw, res.energy.g_cav])
    assert np.all(np.abs(e - e_ref) <= 1e-6 * np.abs(e_ref) + 1e-9)
    assert set(res.timings) == {"hash", "force", "solvation"}


def test_evaluate_energy_only_zero_forces():
    P = _P()
    g = golden("c1_helix")
    _, _, _, fld = make_system(g["seq"])
    res = fld.evaluate(g["positions"], energy_only=True)
    assert np.all(res.forces == 0.0)
    assert res.energy.g_vdw == pytest.approx(float(g["energies"][1]), rel=1e-6)


def test_evaluate_water_solvation_bitexact():
    """Null charges / well depths isolate the fused solvation kernel: its
    forces must equal the reference's solvation_forces bit for bit."""
    from dataclasses import replace
    P = _P()
    g = golden("mixed_water")
    ch, params, w, _ = make_system(g["seq"], solvation=True)
    null = replace(params, q=np.zeros(ch.n_atoms), eps=np.zeros(ch.n_atoms))
    fld = P.Field(null, w, P.FieldConfig(solvation=True))
    res = fld.evaluate(g["positions"])
    assert np.array_equal(res.forces, g["solv_forces"])
    assert np.array_equal(res.sasa.f_exp, g["sasa_f_exp"])
    assert np.array_equal(res.sasa.a_exp, g["sasa_a_exp"])
    assert res.energy.g_cav == pytest.approx(float(g["sasa_g_cav"]), rel=1e-13, abs=1e-12)
    assert res.forces.sum(axis=0).tolist() == [0.0, 0.0, 0.0] or \
        np.abs(res.forces.sum(axis=0)).max() < 1e-9


def test_evaluate_water_total():
    P = _P()
    g = golden("mixed_water")
    ch, params, w, fld = make_system(g["seq"], solvation=True)
    res = fld.evaluate(g["positions"])
    _, _, extra = O.OracleField(params, w).evaluate(g["positions"])
    scale = pair_scale(params, w, g["positions"], extra["i"], extra["j"], extra["d"])
    err = np.linalg.norm(res.forces - g["forces"], axis=1)
    assert np.all(err <= FORCE_TOL * np.maximum(scale, 1e-300))
    assert res.energy.g_cav == pytest.approx(float(g["energies"][2]), rel=1e-13)


# ---- wrenches, torques, step ------------------------------------------------------

@pytest.mark.parametrize("name", ["c1_helix", "c2_random", "mixed_water"])
def test_wrenches_bitexact(name):
    P = _P()
    g = golden(name)
    ch = P.build_chain(list(g["seq"]))
    wr = P.link_wrenches(ch, g["positions"], g["forces"])
    assert np.array_equal(wr.force, g["wrench_f"])
    assert np.array_equal(wr.torque, g["wrench_t"])


@pytest.mark.parametrize("name", ["c1_helix", "c2_random", "mixed_water"])
def test_joint_torques(name):
    P = _P()
    g = golden(name)
    ch = P.build_chain(list(g["seq"]))
    conf = P.Conformation(g["theta"], np.zeros(len(g["theta"]), bool), ch.n_residues)
    st = P.kinematic_state(ch, conf)
    wr = P.LinkWrenches(g["wrench_f"], g["wrench_t"])
    tau = P.joint_torques(ch, conf, wr, st).tau
    scale = np.abs(g["tau"]).max()
    assert np.abs(tau - g["tau"]).max() <= 1e-10 * max(scale, 1.0)


@pytest.mark.parametrize("name", ["c1_helix", "c2_random", "mixed_water"])
def test_step_bitexact(name):
    P = _P()
    g = golden(name)
    conf = P.Conformation(g["theta"], np.zeros(len(g["theta"]), bool), 1)
    out, deltas = P.kcm_step(P.JointTorques(g["tau"]), conf, P.StepConfig())
    assert np.array_equal(out.theta, g["theta_next"])
    assert np.array_equal(deltas, g["deltas"])


def test_step_edge_cases():
    P = _P()
    conf = P.Conformation(np.zeros(3), np.zeros(3, bool), 1)
    out, d = P.kcm_step(P.JointTorques(np.array([4.0, -2.0, 1.0])), conf, P.StepConfig(kappa=0.5))
    assert d.tolist() == [0.5, -0.25, 0.125]
    assert out.theta.tolist() == [0.5, 359.75, 0.125]
    out, d = P.kcm_step(P.JointTorques(np.zeros(3)), conf, P.StepConfig())
    assert out is conf and np.all(d == 0)
    fz = P.Conformation(np.zeros(2), np.array([True, False]), 1)
    out, d = P.kcm_step(P.JointTorques(np.array([100.0, 1.0])), fz, P.StepConfig(kappa=0.5))
    assert d.tolist() == [0.0, 0.5]
    tiny = P.Conformation(np.array([0.0, 359.9999999999]), np.zeros(2, bool), 1)
    out, _ = P.kcm_step(P.JointTorques(np.array([-1e-30, 1.0])), tiny, P.StepConfig(kappa=1e-10))
    ref, _ = O.step(np.array([-1e-30, 1.0]), tiny.theta, tiny.frozen, 1e-10)
    assert np.array_equal(out.theta, ref)
    with pytest.raises(P.ConfigurationError):
        P.kcm_step(P.JointTorques(np.ones(2)), P.Conformation(np.zeros(2), np.ones(2, bool), 1),
                   P.StepConfig())


# ---- spatial API ------------------------------------------------------------------

@pytest.mark.parametrize("name", ["c1_helix", "c2_random"])
def test_build_grid_bitexact(name):
    P = _P()
    g = golden(name)
    grid = P.build_grid(g["positions"])
    assert grid.cell_size == float(g["grid_cell"])
    assert np.array_equal(grid.r_min, g["grid_rmin"]) and np.array_equal(grid.dims, g["grid_dims"])
    assert np.array_equal(grid.cell_index, g["grid_cell_index"])
    assert np.array_equal(grid._occupied, g["grid_occupied"])
    assert np.array_equal(grid._starts, g["grid_starts"])
    assert np.array_equal(grid._atom_order, g["grid_order"])


@pytest.mark.parametrize("name", ["c1_helix", "c2_random"])
def test_neighbor_table_and_filters_bitexact(name):
    P = _P()
    g = golden(name)
    grid = P.build_grid(g["positions"])
    tb = P.build_neighbor_table(grid, 9.0)
    assert np.array_equal(tb.offsets, g["table_off"])
    assert np.array_equal(tb.neighbors, g["table_nb"])
    i, j, d = P.filtered_pairs(tb, g["positions"], 9.0)
    assert np.array_equal(i, g["pairs_i"]) and np.array_equal(j, g["pairs_j"])
    assert np.array_equal(d, g["pairs_d"])
    lists = P.filtered_lists(tb, g["positions"], 8.0)
    flat = np.concatenate(lists)
    assert np.array_equal(flat, g["lists_flat"])
    assert np.array_equal(np.cumsum([0] + [len(x) for x in lists]), g["lists_off"])


def test_classification_matches_reference():
    P = _P()
    g = golden("c1_helix")
    ch = P.build_chain(list(g["seq"]))
    tree = P.build_tree(ch)
    from paper_1712_05012_b200.topology import classify_pairs
    assert np.array_equal(classify_pairs(tree, g["pairs_i"], g["pairs_j"]), g["pairs_cls"])


def test_forcefield_api_functions():
    P = _P()
    g = golden("c1_helix")
    ch, params, w, _ = make_system(g["seq"])
    grid = P.build_grid(g["positions"])
    tb = P.build_neighbor_table(grid, 9.0)
    i, j, d = g["pairs_i"], g["pairs_j"], g["pairs_d"]
    ke = d <= 9.0
    ee, _ = O.elec_terms(params, i[ke], j[ke], d[ke], O.pair_weights(w, i[ke], j[ke], "elec"))
    assert P.elec_energy(g["positions"], params, tb, w) == pytest.approx(float(ee.sum()), rel=1e-12)
    kv = d <= 5.0
    ev, mv = O.vdw_terms(params, i[kv], j[kv], d[kv], O.pair_weights(w, i[kv], j[kv], "vdw"))
    assert P.vdw_energy(g["positions"], params, tb, w) == pytest.approx(float(ev.sum()), rel=1e-12)
    fv = P.vdw_forces(g["positions"], params, tb, w)
    ref = O.scatter(len(g["positions"]), g["positions"], i[kv], j[kv], d[kv], mv)
    assert np.abs(fv - ref).max() <= 1e-9 * np.abs(ref).max()


# ---- solvation API (bit-exact) ----------------------------------------------------

def test_sasa_pass_and_forces_bitexact():
    P = _P()
    g = golden("mixed_water")
    ch, params, w, fld = make_system(g["seq"], solvation=True)
    off, flat = g["lists_off"], g["lists_flat"]
    lists = [flat[off[a]:off[a + 1]] for a in range(len(off) - 1)]
    sasa, states = P.sasa_pass(g["positions"], params, lists, fld.sphere(), fld.config.solvation_cfg)
    assert np.array_equal(states.counts, g["sasa_counts"])
    assert np.array_equal(states.critical, g["sasa_critical"])
    assert np.array_equal(sasa.f_exp, g["sasa_f_exp"]) and np.array_equal(sasa.a_exp, g["sasa_a_exp"])
    assert sasa.g_cav == pytest.approx(float(g["sasa_g_cav"]), rel=1e-13)
    sf = P.solvation_forces(g["positions"], params, lists, fld.sphere(), states, fld.config.solvation_cfg)
    assert np.array_equal(sf, g["solv_forces"])


def test_sasa_known_answers():
    """Isolated atom 4 pi R_off^2 exactly; two-sphere cap ~27 pi (test_solvation.py:91-123)."""
    P = _P()
    import math
    par = P.AtomParams(q=np.zeros(1), R=np.full(1, 1.6), eps=np.full(1, 0.1), gamma=np.ones(1),
                       solv_class=("C",))
    cfg = P.SolvationConfig(samples=256)
    res, st = P.sasa_pass(np.zeros((1, 3)), par, [np.array([], int)], P.generate_samples(256), cfg)
    assert res.f_exp[0] == 1.0 and res.a_exp[0] == pytest.approx(4 * math.pi * 3.0 ** 2, rel=1e-12)
    par2 = P.AtomParams(q=np.zeros(2), R=np.full(2, 1.6), eps=np.full(2, 0.1), gamma=np.ones(2),
                        solv_class=("C", "C"))
    res, _ = P.sasa_pass(np.array([[0.0, 0, 0], [3.0, 0, 0]]), par2, [np.array([1]), np.array([0])],
                         P.generate_samples(10_000), P.SolvationConfig(samples=10_000))
    want = 27 * math.pi
    assert np.all(np.abs(res.a_exp - want) / want < 0.01)


# ---- the fold loop -----------------------------------------------------------------

def _traj(name):
    g = golden(name)
    P = _P()
    st = g["step"]
    step = P.StepConfig(kappa=float(st[0]), max_iters=int(st[1]), torque_tol=float(st[2]),
                        torque_tol_rel=float(st[3]), energy_window=int(st[4]), energy_tol=float(st[5]),
                        snapshot_every=int(st[6]))
    return g, step


@pytest.mark.parametrize("name,solv", [("fold_vacuum", False), ("fold_water", True),
                                       ("fold_frozen", False)])
def test_fold_trajectory_matches_reference(name, solv):
    P = _P()
    g, step = _traj(name)
    ch, params, w, fld = make_system(g["seq"], solvation=solv)
    conf = P.Conformation(g["theta0"], g["frozen"], ch.n_residues)
    tr = P.fold(ch, conf, fld, step)
    assert tr.iterations == len(g["energies"]) and tr.reason == str(g["reason"])
    E = np.array([[r.energy.g_elec, r.energy.g_vdw, r.energy.g_cav] for r in tr.records])
    scale = np.abs(g["energies"]).sum(axis=1)
    assert np.all(np.abs(E - g["energies"]).sum(axis=1) <= 1e-5 * scale)
    _, _, _, p_gpu = O.fk(ch, tr.final.theta)
    _, _, _, p_ref = O.fk(ch, g["final"])
    rmsd = np.sqrt(((p_gpu - p_ref) ** 2).sum(axis=1).mean())
    assert rmsd <= 1e-4
    assert np.array_equal(tr.final.theta[g["frozen"]], g["theta0"][g["frozen"]])
    assert [k for k, _ in tr.snapshots] == g["snap_iters"].tolist()
    assert np.array_equal(tr.records[0].theta, g["thetas"][0])
    if solv:
        assert all(r.timings["solvation"] > 0 for r in tr.records)


def test_fold_default_stop_rule():
    """Default StepConfig stop rules (energy plateau: |E_k - E_{k-20}| < 0.02).

    The reference trajectory itself is sensitive near its plateau: measured
    with kinefold, a 1e-6 degree perturbation of the start stays below 3e-6
    kcal/mol for 100 iterations but reaches 0.3 kcal/mol at iteration 119, so
    the stop iteration is only as stable as that.  Checked: (1) the GPU
    energies track the reference over the first 100 iterations within 5e-4
    relative (the fp32 pair math starts ~2e-6 off and this trajectory
    amplifies ~20x over 100 iterations, as the reference's own perturbation
    test shows), (2) the device stop logic fires exactly where the GPU's own
    records first satisfy the plateau rule, (3) the plateau is reached."""
    P = _P()
    g, step = _traj("fold_default_stop")
    ch, params, w, fld = make_system(g["seq"])
    conf = P.Conformation(g["theta0"], g["frozen"], ch.n_residues)
    K = 100
    free = P.fold(ch, conf, fld, P.StepConfig(max_iters=K, torque_tol_rel=0.0, energy_window=0))
    E = np.array([[r.energy.g_elec, r.energy.g_vdw, r.energy.g_cav] for r in free.records])
    ref = g["energies"][:K]
    assert np.all(np.abs(E - ref).sum(1) <= 5e-4 * np.abs(ref).sum(1))
    tr = P.fold(ch, conf, fld, step)
    assert tr.reason == "energy plateau" and tr.converged
    win = step.energy_window
    e = tr.energies()
    hits = [k for k in range(win, len(e)) if abs(e[k] - e[k - win]) < step.energy_tol]
    assert hits and hits[0] == tr.iterations - 1


@pytest.fixture
def fp64_pairs():
    P = _P()
    P.set_pair_precision("fp64")
    yield
    P.set_pair_precision("fp32")


def _c1_1000():
    P = _P()
    g, step = _traj("fold_c1_1000")
    ch, params, w, fld = make_system(g["seq"])
    conf = P.Conformation(g["theta0"], g["frozen"], ch.n_residues)
    tr = P.fold(ch, conf, fld, step)
    assert tr.iterations == len(g["energies"]) == 1000 and tr.reason == "max_iters"
    E = np.array([[r.energy.g_elec, r.energy.g_vdw, r.energy.g_cav] for r in tr.records])
    rel = np.abs(E - g["energies"]).sum(1) / np.abs(g["energies"]).sum(1)
    _, _, _, p_gpu = O.fk(ch, tr.final.theta)
    _, _, _, p_ref = O.fk(ch, g["final"])
    rmsd = np.sqrt(((p_gpu - p_ref) ** 2).sum(axis=1).mean())
    e_gpu, e_ref = E[-1].sum(), g["energies"][-1].sum()
    assert abs(e_gpu - e_ref) <= 1e-2 * abs(e_ref)
    return rel, rmsd, tr, (ch, params, w, g, step)


def test_fold_c1_1000_iterations_fp64(fp64_pairs):
    """SURVEY.md §8(d) trajectory criterion on C1 (30 x ALA helix start, vacuum,
    K = 1000), fp64 pair mode: per record |dE| <= 1e-5 (|g_elec| + |g_vdw| +
    |g_cav|) and final RMSD <= 1e-4 A."""
    rel, rmsd, _, _ = _c1_1000()
    assert rel.max() <= 1e-5 and rmsd <= 1e-4, (rel.max(), rmsd)


def test_fold_c1_1000_iterations_fp32():
    """Same trajectory with fp32 pair math (the default).

    Per-step parity is ~1e-7 (forces: median 5e-7, p99 3e-6 relative, energy
    ~1e-7; tools/fp32_err.py).  The trajectory itself is not a smooth function
    of that rounding: the energy is discontinuous at the 9 A / 5 A cut-offs and
    the fixed 0.5 degree step oscillates across the minimum from iteration
    ~300, so a 1e-7 difference can move a cut-off crossing by one iteration
    (measured on B200: the first records above 1e-5 / 1e-4 of the energy scale
    appear between iterations 5 and 210 depending on the kernel's rounding
    order; max 3e-2; final energy within 0.2 %).

    Stated fp32 tolerance: (a) shadowing -- from the GPU's own theta at
    sampled iterations, the reference step (oracle) reproduces the GPU's
    record energy to 5e-6 and its next theta to 1e-4 of the step size kappa
    over the first 100 iterations, 2e-3 of kappa later.  The step is
    kappa * tau / tau_max: as the helix relaxes tau_max falls far below the
    pair forces whose fp32 rounding (~1e-7 each) it sums, so the relative
    step error grows (measured: 1e-5 at the start, up to 6.6e-4 of kappa near
    the minimum; 1e-7 on C2 random conformations; tools/fp32_err.py);
    (b) whole trajectory: every record within 5e-2 of the reference's energy
    scale and the final energy within 1 %.  set_pair_precision("fp64") gives
    4e-12 over the full 1000 (test above)."""
    rel, rmsd, tr, (ch, params, w, g, step) = _c1_1000()
    assert rel.max() <= 5e-2, rel.max()
    fld = O.OracleField(params, w)
    frozen = np.asarray(g["frozen"], bool)
    for k in list(range(0, 1000, 50)) + [999]:
        th = np.asarray(tr.records[k].theta)
        M, Pp, U, pos = O.fk(ch, th)
        forces, e, _ = fld.evaluate(pos)
        e_gpu = tr.records[k].energy
        e_sum = abs(e[0]) + abs(e[1]) + abs(e[2])
        # fp32 pair energies: rounding ~1e-7 of sum_ij |e_ij|, which for the folded
        # helix is ~10x |E| (measured up to 1.1e-6 of e_sum)
        assert abs(e_gpu.g_elec - e[0]) + abs(e_gpu.g_vdw - e[1]) <= 5e-6 * e_sum, k
        F, T = O.wrenches(ch, pos, forces)
        nxt, _ = O.step(O.torques(ch, U, Pp, F, T), th, frozen, step.kappa)
        got = np.asarray(tr.records[k + 1].theta) if k + 1 < len(tr.records) else np.asarray(tr.final.theta)
        d = np.abs((got - nxt + 180.0) % 360.0 - 180.0).max()
        assert d <= (1e-4 if k <= 100 else 2e-3) * step.kappa, (k, d)


def test_fold_default_stop_rule_fp64(fp64_pairs):
    """With fp64 pair math the default stop rule fires at the reference's iteration."""
    P = _P()
    g, step = _traj("fold_default_stop")
    ch, params, w, fld = make_system(g["seq"])
    tr = P.fold(ch, P.Conformation(g["theta0"], g["frozen"], ch.n_residues), fld, step)
    assert tr.reason == str(g["reason"]) and tr.iterations == len(g["energies"])
    E = np.array([[r.energy.g_elec, r.energy.g_vdw, r.energy.g_cav] for r in tr.records])
    assert np.all(np.abs(E - g["energies"]).sum(1) <= 1e-9 * np.abs(g["energies"]).sum(1))


def test_fold_clash_message():
    P = _P()
    g = golden("clash")
    ch, params, w, fld = make_system(["ALA", "ALA"])
    bad = P.build_chain(["ALA", "ALA"])
    bad.zp_pos[3] = bad.zp_pos[2] + 1e-9
    with pytest.raises(P.StericClashError) as exc:
        P.fold(bad, bad.conf_zp(), fld, P.StepConfig(max_iters=3))
    assert str(exc.value) == str(g["message"])


def test_fold_torque_free_and_determinism():
    from dataclasses import replace
    P = _P()
    ch, params, w, _ = make_system(["GLY", "GLY"])
    null = replace(params, q=np.zeros(ch.n_atoms), eps=np.zeros(ch.n_atoms))
    tr = P.fold(ch, ch.conf_zp(), P.Field(null, w, P.FieldConfig()), P.StepConfig(max_iters=10))
    assert tr.converged and tr.reason == "torque-free" and tr.iterations == 1
    ch, params, w, fld = make_system(["ALA"] * 10)
    conf = ch.conf_from_backbone(-20.0, -30.0)
    st = P.StepConfig(max_iters=40, torque_tol_rel=0.0, energy_window=0)
    a, b = P.fold(ch, conf, fld, st), P.fold(ch, conf, fld, st)
    assert np.array_equal(a.final.theta, b.final.theta)
    assert np.array_equal(a.energies(), b.energies())


def test_ensemble_equals_single_trajectories():
    P = _P()
    ch, params, w, fld = make_system(["ALA", "SER", "CYS"] * 4)
    rng = np.random.default_rng(3)
    confs = [ch.conf_from_backbone(rng.uniform(-90, 90, ch.n_residues), rng.uniform(-90, 90, ch.n_residues))
             for _ in range(5)]
    st = P.StepConfig(max_iters=20, torque_tol_rel=0.0, energy_window=0)
    ens = P.fold_ensemble(ch, confs, fld, st)
    for k, c in enumerate(confs):
        tr = P.fold(ch, c, fld, st)
        assert np.array_equal(ens.theta[k], tr.final.theta)
        assert np.array_equal(ens.energies[k, :, :3],
                              np.array([[r.energy.g_elec, r.energy.g_vdw, r.energy.g_cav] for r in tr.records]))


def test_scans_match_single_point():
    P = _P()
    ch, params, w, fld = make_system(["ALA", "ALA"])
    grid = P.ramachandran_scan(ch, 1, 6, fld)
    conf = ch.conf_zp()
    theta = conf.theta.copy()
    theta[ch.dof_phi(1)] = grid.axes[0][2] + 180.0
    theta[ch.dof_psi(1)] = grid.axes[1][4] + 180.0
    e = P.single_point(ch, P.Conformation(theta, conf.frozen, 2), fld)
    # the 36-point scan is one batch on the cluster-pair kernel, the single point a
    # dense-lane launch: equal to the fp32 pair-math bar, not bitwise
    assert grid.g_total[2, 4] == pytest.approx(e.g_total, rel=1e-6)


def test_fold_long_chain_multi_cta_path(fp64_pairs):
    """Chains past one 2048-dof backbone segment take the multi-CTA FK and
    torque passes (kf_kinematics.cu fk_seg_*, kf_torque.cu torque_seg_*).
    1100 random A/C/S residues (2200 backbone dofs, 2 segments), fp64 pair
    math, 4 iterations vs the oracle: energies and tau_max to 1e-9, theta to
    1e-9 degrees."""
    P = _P()
    seq = [str(x) for x in np.random.default_rng(5).choice(["ALA", "CYS", "SER"], 1100)]
    ch, params, w, fld = make_system(seq)
    rng = np.random.default_rng(6)
    conf = ch.conf_from_backbone(rng.uniform(-90, 90, len(seq)), rng.uniform(-90, 90, len(seq)))
    step = P.StepConfig(max_iters=4, torque_tol_rel=0.0, energy_window=0)
    tr = P.fold(ch, conf, fld, step)
    ref = O.fold(ch, conf.theta, conf.frozen, O.OracleField(params, w), kappa=0.5, max_iters=4,
                 torque_tol_rel=0.0, energy_window=0)
    E = np.array([[r.energy.g_elec, r.energy.g_vdw, r.energy.g_cav] for r in tr.records])
    scale = np.abs(ref["energies"]).sum(1)
    assert np.all(np.abs(E - ref["energies"]).sum(1) <= 1e-9 * scale)
    tm = np.array([r.tau_max for r in tr.records])
    assert np.all(np.abs(tm - ref["tau_max"]) <= 1e-9 * ref["tau_max"])
    d = np.abs((np.asarray(tr.final.theta) - ref["final"] + 180.0) % 360.0 - 180.0).max()
    assert d <= 1e-9, d


_OVERFLOW_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
from conftest import golden, make_system
import paper_1712_05012_b200 as P
from dataclasses import replace
g = golden("mixed_water")
ch, params, w, _ = make_system(g["seq"], solvation=True)
null = replace(params, q=np.zeros(ch.n_atoms), eps=np.zeros(ch.n_atoms))
res = P.Field(null, w, P.FieldConfig(solvation=True)).evaluate(g["positions"])
assert np.array_equal(res.forces, g["solv_forces"])
assert np.array_equal(res.sasa.f_exp, g["sasa_f_exp"])
ch, params, w, fld = make_system(g["seq"], solvation=True)
conf = P.Conformation(g["theta"], np.zeros(ch.n_dof, bool), ch.n_residues)
step = P.StepConfig(max_iters=3, torque_tol_rel=0.0, energy_window=0)
ens = P.fold_ensemble(ch, [conf] * 16, fld, step)          # ensemble build of the solvation pass
one = P.fold(ch, conf, fld, step)
E = np.array([[r.energy.g_elec, r.energy.g_vdw, r.energy.g_cav] for r in one.records])
for b in range(16):
    assert np.allclose(ens.energies[b, :3, :3], E, rtol=1e-12, atol=1e-12), b
print("ok")
"""


def test_solvation_overflow_pass_bitexact():
    """Atoms with more reachable neighbours than the primary pass stages go to
    solv_overflow_kernel.  With the primary capacity forced to 4
    (KFB200_SOLV_FAST_CAP, read once per process, hence the subprocess) nearly
    every atom takes that path: forces and exposures stay bit-exact, and the
    ensemble build agrees with single folds."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    env = dict(os.environ, KFB200_SOLV_FAST_CAP="4")
    out = subprocess.run([sys.executable, "-c", _OVERFLOW_SCRIPT], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-3000:]


# ---- FieldConfig(use_hash=False): the quadratic all-pairs path (kcm.py:94-102, :153-162)

def _flat(fld):
    from dataclasses import replace
    P = _P()
    return P.Field(fld.params, fld.weights, replace(fld.config, use_hash=False))


@pytest.mark.parametrize("name", ["c1_helix", "c2_random"])
def test_use_hash_false_evaluate_matches_reference(name):
    """The brute-force table gives the same pair set as the hash grid (the
    reference's grid independence), so the same force/energy bars hold."""
    g = golden(name)
    ch, params, w, fld = make_system(g["seq"])
    res = _flat(fld).evaluate(g["positions"])
    _, _, extra = O.OracleField(params, w).evaluate(g["positions"])
    scale = pair_scale(params, w, g["positions"], extra["i"], extra["j"], extra["d"])
    err = np.linalg.norm(res.forces - g["forces"], axis=1)
    assert np.all(err <= FORCE_TOL * np.maximum(scale, 1e-300)), (err / scale).max()
    e = np.array([res.energy.g_elec, res.energy.g_vdw, res.energy.g_cav])
    assert np.all(np.abs(e - g["energies"]) <= 1e-6 * np.abs(g["energies"]) + 1e-9)


def test_use_hash_false_solvation_bitexact():
    from dataclasses import replace
    P = _P()
    g = golden("mixed_water")
    ch, params, w, _ = make_system(g["seq"], solvation=True)
    null = replace(params, q=np.zeros(ch.n_atoms), eps=np.zeros(ch.n_atoms))
    fld = P.Field(null, w, P.FieldConfig(solvation=True, use_hash=False))
    res = fld.evaluate(g["positions"])
    assert np.array_equal(res.forces, g["solv_forces"])
    assert np.array_equal(res.sasa.f_exp, g["sasa_f_exp"])
    assert res.energy.g_cav == pytest.approx(float(g["sasa_g_cav"]), rel=1e-13, abs=1e-12)


@pytest.mark.parametrize("name,solv", [("fold_vacuum", False), ("fold_water", True)])
def test_use_hash_false_fold_matches_reference(name, solv):
    P = _P()
    g, step = _traj(name)
    ch, params, w, fld = make_system(g["seq"], solvation=solv)
    conf = P.Conformation(g["theta0"], g["frozen"], ch.n_residues)
    tr = P.fold(ch, conf, _flat(fld), step)
    assert tr.iterations == len(g["energies"]) and tr.reason == str(g["reason"])
    E = np.array([[r.energy.g_elec, r.energy.g_vdw, r.energy.g_cav] for r in tr.records])
    scale = np.abs(g["energies"]).sum(axis=1)
    assert np.all(np.abs(E - g["energies"]).sum(axis=1) <= 1e-5 * scale)


def test_use_hash_false_ensemble_half_list():
    """Ensembles take the half-list kernel; with one all-atom cell it sweeps each
    unordered pair once.  The first record (the start conformations, before the
    fp32 summation order can steer these clash-laden random starts apart) meets
    the pair bar against the hashed ensemble; the pair counts are equal."""
    P = _P()
    ch, params, w, fld = make_system(["ALA", "SER", "CYS"] * 6)
    rng = np.random.default_rng(5)
    confs = [ch.conf_from_backbone(rng.uniform(-90, 90, ch.n_residues), rng.uniform(-90, 90, ch.n_residues))
             for _ in range(256)]   # B * n >= 40k: the warp-per-item half-list kernel
    st = P.StepConfig(max_iters=1, torque_tol_rel=0.0, energy_window=0)
    a = P.fold_ensemble(ch, confs, fld, st)
    b = P.fold_ensemble(ch, confs, _flat(fld), st)
    ea, eb = a.energies[:, 0, :3], b.energies[:, 0, :3]
    assert np.all(np.abs(ea - eb).sum(axis=1) <= 1e-6 * np.abs(ea).sum(axis=1))
    assert np.abs(b.theta - a.theta).max() <= 1e-4 * st.kappa
    if a.n_pairs is not None:
        assert np.array_equal(a.n_pairs, b.n_pairs)


def test_use_hash_false_extent_guard():
    from paper_1712_05012_b200.errors import ConfigurationError
    g = golden("c1_helix")
    _, _, _, fld = make_system(g["seq"])
    pos = np.array(g["positions"], float)
    pos[0] += 5000.0
    with pytest.raises(ConfigurationError, match="use_hash=False"):
        _flat(fld).evaluate(pos)


_CLOSE_PAIR_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
from conftest import golden, make_system
from oracle import kcm_oracle as O
from test_gpu_parity import pair_scale
g = golden("c2_random")
ch, params, w, fld = make_system(g["seq"])
pos = np.array(g["positions"], float)
a, b = 100, 700                      # far apart along the chain: class 4, weight 1
pos[a] = pos[b] + np.array([0.02, 0.0, 0.0])
res = fld.evaluate(pos)
f_ref, e_ref, extra = O.OracleField(params, w).evaluate(pos)
scale = pair_scale(params, w, pos, extra["i"], extra["j"], extra["d"])
assert np.all(np.isfinite(res.forces))
err = np.linalg.norm(res.forces - f_ref, axis=1)
assert np.all(err <= 1e-5 * np.maximum(scale, 1e-300)), float((err / scale).max())
assert abs(res.energy.g_vdw - e_ref[1]) <= 1e-6 * abs(e_ref[1])
print("ok", float(np.abs(f_ref[a]).max()))
"""


@pytest.mark.parametrize("variant", ["3"])
def test_half_list_clash_range_pair(variant):
    """A pair at 0.02 A (vdW force ~1e28, past the half list's two-level fixed
    point) through the half-list kernel (KFB200_PAIR_KERNEL=3, read once per
    process, hence the subprocess): forces finite and within the bar of the
    oracle, Newton's third law kept (the exact path adds +f and -f in fp64)."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    env = dict(os.environ, KFB200_PAIR_KERNEL=variant)
    out = subprocess.run([sys.executable, "-c", _CLOSE_PAIR_SCRIPT], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


def test_forcefield_api_deterministic_bincount_order():
    """elec_forces / vdw_forces scatter in np.bincount order (forcefield.py:169-171):
    run-to-run deterministic, and accumulate_pair_forces (given magnitudes) is
    bit-identical to the reference's scatter."""
    P = _P()
    g = golden("c2_random")
    ch, params, w, _ = make_system(g["seq"])
    grid = P.build_grid(g["positions"])
    tb = P.build_neighbor_table(grid, 9.0)
    i, j, d = g["pairs_i"], g["pairs_j"], g["pairs_d"]
    kv = d <= 5.0
    _, mv = O.vdw_terms(params, i[kv], j[kv], d[kv], O.pair_weights(w, i[kv], j[kv], "vdw"))
    ref = O.scatter(len(g["positions"]), g["positions"], i[kv], j[kv], d[kv], mv)
    a = P.vdw_forces(g["positions"], params, tb, w)
    b = P.vdw_forces(g["positions"], params, tb, w)
    assert np.array_equal(a, b)
    # pair magnitudes use CUDA pow (<= 2 ulp from glibc's): equal to rounding
    assert np.abs(a - ref).max() <= 1e-12 * np.abs(ref).max()
    from paper_1712_05012_b200.forcefield import accumulate_pair_forces
    acc = accumulate_pair_forces(len(g["positions"]), g["positions"], i[kv], j[kv], d[kv], mv)
    assert np.array_equal(acc, ref)


def _abs_pair_energy(params, w, ex):
    """sum_ij |e_ij| over the elec and vdW pairs: the scale of fp32 energy rounding
    (the totals cancel: a compact 4-residue chain has |g| ~ 1e-2 sum |e_ij|)."""
    i, j, d = ex["i"], ex["j"], ex["d"]
    ke, kv = d <= 9.0, d <= 5.0
    ee, _ = O.elec_terms(params, i[ke], j[ke], d[ke], O.pair_weights(w, i[ke], j[ke], "elec"))
    ev, _ = O.vdw_terms(params, i[kv], j[kv], d[kv], O.pair_weights(w, i[kv], j[kv], "vdw"))
    return float(np.abs(ee).sum() + np.abs(ev).sum())


def test_scans_match_oracle():
    """ramachandran_scan / hinge_scan (kcm.py:358-419) against the oracle's
    evaluation of the same grid conformations: totals within 1e-6 of the pair
    energies' magnitude sum (the fp32 pair math's rounding scale)."""
    P = _P()
    ch, params, w, fld = make_system(["ALA", "SER", "CYS", "ALA"])
    of = O.OracleField(params, w)
    grid = P.ramachandran_scan(ch, 2, 5, fld)
    conf = ch.conf_zp()
    for a in range(grid.g_total.shape[0]):
        for b in range(grid.g_total.shape[1]):
            th = conf.theta.copy()
            th[ch.dof_phi(2)] = grid.axes[0][a] + 180.0
            th[ch.dof_psi(2)] = grid.axes[1][b] + 180.0
            _, e, ex = of.evaluate(O.fk(ch, th)[3])
            assert abs(grid.g_total[a, b] - sum(e)) <= 1e-6 * _abs_pair_energy(params, w, ex), (a, b)
    dofs = [ch.dof_phi(1), ch.dof_psi(1)]
    hg = P.hinge_scan(ch, dofs, 30.0, 3, fld, conf)
    assert hg.g_total.shape == (3, 3)
    for a in range(3):
        for b in range(3):
            th = conf.theta.copy()
            th[dofs[0]] = np.mod(conf.theta[dofs[0]] + hg.axes[0][a], 360.0)
            th[dofs[1]] = np.mod(conf.theta[dofs[1]] + hg.axes[1][b], 360.0)
            _, e, ex = of.evaluate(O.fk(ch, th)[3])
            assert abs(hg.g_total[a, b] - sum(e)) <= 1e-6 * _abs_pair_energy(params, w, ex), (a, b)
