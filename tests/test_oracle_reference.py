"""Oracle vs the live reference package on random systems (build container
only: skipped where /root/reference is absent, e.g. on the GPU box)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from oracle import kcm_oracle as O

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


@pytest.fixture(scope="module")
def K():
    sys.path.insert(0, REF)
    import kinefold
    return kinefold


def _system(K, seq, **cfg):
    ch = K.build_chain(seq)
    ps = K.load_params()
    p = ps.resolve(ch)
    w = K.TreeWeights(K.build_tree(ch), ps.weights)
    return ch, p, w, K.Field(p, w, K.FieldConfig(**cfg))


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_oracle_matches_reference_random_systems(K, seed):
    rng = np.random.default_rng(seed)
    seq = list(rng.choice(["ALA", "CYS", "SER", "GLY"], int(rng.integers(3, 25))))
    ch, p, w, fld = _system(K, seq)
    conf = ch.conf_from_backbone(rng.uniform(-180, 180, len(seq)), rng.uniform(-180, 180, len(seq)))
    st = K.kinematic_state(ch, conf)
    _, _, _, pos = O.fk(ch, conf.theta)
    assert np.array_equal(pos, st.positions)
    try:
        r = fld.evaluate(st.positions)
    except K.KinefoldError:
        with pytest.raises(O.OracleError):
            O.OracleField(p, w).evaluate(pos)
        return
    f, e, _ = O.OracleField(p, w).evaluate(pos)
    assert np.array_equal(f, r.forces)
    assert e == (r.energy.g_elec, r.energy.g_vdw, r.energy.g_cav)


def test_oracle_matches_reference_uniform_weights_and_alpha(K):
    rng = np.random.default_rng(9)
    pos = rng.uniform(0, 12, size=(60, 3))
    n = len(pos)
    params = K.AtomParams(q=rng.normal(0, 0.3, n), R=rng.uniform(1.0, 2.0, n), eps=rng.uniform(0.01, 0.2, n),
                          gamma=np.zeros(n), solv_class=("C",) * n)
    for alpha in (0.05, 1.0, 5.0):
        g = K.build_grid(pos, K.GridConfig(alpha=alpha))
        og = O.grid(pos, alpha)
        assert np.array_equal(g._atom_order, og["order"]) and g.cell_size == og["cell"]
        tb = K.build_neighbor_table(g, 9.0)
        off, flat = O.neighbor_table(og, 9.0)
        assert np.array_equal(tb.neighbors, flat) and np.array_equal(tb.offsets, off)
    fld = K.Field(params, K.UniformWeights(0.7), K.FieldConfig())
    r = fld.evaluate(pos)
    f, e, _ = O.OracleField(params, K.UniformWeights(0.7)).evaluate(pos)
    assert np.array_equal(f, r.forces) and e[:2] == (r.energy.g_elec, r.energy.g_vdw)
