"""Generate the golden vectors from the REAL reference package.

Run in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array saved here is an output of ``kinefold`` 0.1.0 itself (the
reference), on inputs built by the reference.  The vectors travel with the
repo, so the GPU box (which has no /root/reference) can check the CUDA path
and the oracle against the reference's own numbers.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import kinefold as K  # noqa: E402
from kinefold.errors import StericClashError  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def system(seq, solvation=False, samples=1024, dielectric=None):
    ch = K.build_chain(seq)
    ps = K.load_params()
    params = ps.resolve(ch)
    w = K.TreeWeights(K.build_tree(ch), ps.weights)
    kw = dict(solvation=solvation, solvation_cfg=K.SolvationConfig(samples=samples))
    if dielectric is not None:
        kw["dielectric"] = dielectric
    return ch, params, w, K.Field(params, w, K.FieldConfig(**kw))


def random_conf(ch, seed):
    rng = np.random.default_rng(seed)
    m = ch.n_residues
    phi = rng.uniform(-90.0, 90.0, m)
    psi = rng.uniform(-90.0, 90.0, m)
    return ch.conf_from_backbone(phi, psi)


def snapshot(name, seq, conf, fld, ch, with_table=True):
    st = K.kinematic_state(ch, conf)
    pos = st.positions
    res = fld.evaluate(pos)
    wr = K.link_wrenches(ch, pos, res.forces)
    tau = K.joint_torques(ch, conf, wr, st).tau
    conf2, deltas = K.kcm_step(K.JointTorques(tau), conf, K.StepConfig())
    out = dict(seq=np.array(seq), theta=conf.theta, positions=pos, forces=res.forces,
               energies=np.array([res.energy.g_elec, res.energy.g_vdw, res.energy.g_cav]),
               wrench_f=wr.force, wrench_t=wr.torque, tau=tau, theta_next=conf2.theta, deltas=deltas,
               link_M=np.array(st.transforms), link_P=np.array(st.joint_points),
               link_U=np.array([np.zeros(3) if u is None else u for u in st.axes]))
    g = K.build_grid(pos)
    out.update(grid_cell=np.array(g.cell_size), grid_rmin=g.r_min, grid_rmax=g.r_max, grid_dims=g.dims,
               grid_cell_index=g.cell_index, grid_occupied=g._occupied, grid_starts=g._starts,
               grid_order=g._atom_order)
    if with_table:
        tb = K.build_neighbor_table(g, 9.0)
        i, j, d = K.filtered_pairs(tb, pos, 9.0)
        lists = K.filtered_lists(tb, pos, 8.0)
        out.update(table_off=tb.offsets, table_nb=tb.neighbors, pairs_i=i, pairs_j=j, pairs_d=d,
                   lists_off=np.concatenate([[0], np.cumsum([len(x) for x in lists])]),
                   lists_flat=np.concatenate(lists))
        from kinefold.topology import classify_pairs
        out["pairs_cls"] = classify_pairs(fld.weights.tree, i, j)
    if fld.config.solvation:
        cav = K.filtered_lists(K.build_neighbor_table(g, fld.config.active_cutoff()), pos, 8.0)
        sasa, states = K.sasa_pass(pos, fld.params, cav, fld.sphere(), fld.config.solvation_cfg)
        sf = K.solvation_forces(pos, fld.params, cav, fld.sphere(), states, fld.config.solvation_cfg)
        out.update(sasa_counts=states.counts, sasa_critical=states.critical, sasa_f_exp=sasa.f_exp,
                   sasa_a_exp=sasa.a_exp, sasa_g_cav=np.array(sasa.g_cav), solv_forces=sf)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(name, ch.n_atoms, "atoms", {k: v.shape for k, v in out.items() if hasattr(v, "shape")}.get("forces"))


def trajectory(name, seq, conf, fld, ch, **step_kw):
    tr = K.fold(ch, conf, fld, K.StepConfig(**step_kw))
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"), seq=np.array(seq), theta0=conf.theta, frozen=conf.frozen,
        energies=np.array([[r.energy.g_elec, r.energy.g_vdw, r.energy.g_cav] for r in tr.records]),
        tau_max=np.array([r.tau_max for r in tr.records]),
        thetas=np.array([r.theta for r in tr.records][:60]), final=tr.final.theta,
        reason=np.array(tr.reason), converged=np.array(tr.converged),
        snap_iters=np.array([k for k, _ in tr.snapshots]),
        step=np.array([step_kw.get(k, getattr(K.StepConfig(), k)) for k in
                       ("kappa", "max_iters", "torque_tol", "torque_tol_rel", "energy_window",
                        "energy_tol", "snapshot_every")]))
    print(name, tr.iterations, tr.reason)


def main():
    rng = np.random.default_rng(0)
    # C1 shape: 30 x ALA helix start
    ch, params, w, fld = system(["ALA"] * 30)
    snapshot("c1_helix", ["ALA"] * 30, ch.conf_from_backbone(-10.0, -10.0), fld, ch)
    # C2 shape: 140 random A/C/S, random +-90 start
    seq2 = list(np.random.default_rng(0).choice(["ALA", "CYS", "SER"], 140))
    ch, params, w, fld = system(seq2)
    snapshot("c2_random", seq2, random_conf(ch, 1), fld, ch)
    # mixed residues in water, constant dielectric variant
    seq3 = ["SER", "ALA", "GLY", "CYS", "ALA"] * 3
    ch, params, w, fld = system(seq3, solvation=True)
    snapshot("mixed_water", seq3, random_conf(ch, 2), fld, ch)
    ch, params, w, fld = system(seq3, dielectric=K.DielectricModel(mode="constant", kappa=4.0))
    snapshot("mixed_const_kappa", seq3, random_conf(ch, 3), fld, ch)
    # trajectories
    ch, params, w, fld = system(["ALA"] * 12)
    trajectory("fold_vacuum", ["ALA"] * 12, ch.conf_from_backbone(-10.0, -10.0), fld, ch,
               max_iters=60, torque_tol_rel=0.0, energy_window=0)
    trajectory("fold_default_stop", ["ALA"] * 8, K.build_chain(["ALA"] * 8).conf_from_backbone(-60.0, -45.0),
               system(["ALA"] * 8)[3], K.build_chain(["ALA"] * 8), max_iters=400)
    ch, params, w, fld = system(["ALA"] * 6, solvation=True)
    trajectory("fold_water", ["ALA"] * 6, ch.conf_from_backbone(-30.0, -30.0), fld, ch,
               max_iters=8, torque_tol_rel=0.0, energy_window=0)
    ch, params, w, fld = system(seq3)
    conf = random_conf(ch, 4).freeze([0, 1, 5])
    trajectory("fold_frozen", seq3, conf, fld, ch, max_iters=25, torque_tol_rel=0.0, energy_window=0)
    # C1 trajectory criterion: 1000 vacuum iterations
    ch, params, w, fld = system(["ALA"] * 30)
    trajectory("fold_c1_1000", ["ALA"] * 30, ch.conf_from_backbone(-10.0, -10.0), fld, ch,
               max_iters=1000, torque_tol_rel=0.0, energy_window=0, snapshot_every=0)
    # clash message (test_kcm.py:204-213 pattern)
    ch, params, w, fld = system(["ALA", "ALA"])
    bad = K.build_chain(["ALA", "ALA"])
    bad.zp_pos[3] = bad.zp_pos[2] + 1e-9
    try:
        K.fold(bad, bad.conf_zp(), fld, K.StepConfig(max_iters=3))
    except StericClashError as exc:
        np.savez_compressed(os.path.join(OUT, "clash.npz"), message=np.array(str(exc)),
                            zp_pos=bad.zp_pos)
        print("clash", exc)
    _ = rng


if __name__ == "__main__":
    main()
