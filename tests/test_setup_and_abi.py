"""Host-side checks that need no GPU: setup tables vs the reference's golden
data, the C-ABI library's symbol table and struct layouts, the API surface,
and the no-CPU-fallback contract."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden, have_gpu, make_system
from oracle import kcm_oracle as O

import paper_1712_05012_b200 as P
from paper_1712_05012_b200 import _native as N


# ---- setup tables (host, once per system) are bit-identical to the reference --

@pytest.mark.parametrize("name", ["c1_helix", "c2_random", "mixed_water"])
def test_builder_reproduces_reference_geometry(name):
    """Our canonical builder + the oracle's sequential FK give the reference's
    positions bit for bit, so the chain tables are the reference's."""
    g = golden(name)
    ch = P.build_chain(list(g["seq"]))
    assert ch.n_atoms == len(g["positions"]) and ch.n_dof == len(g["theta"])
    _, _, _, pos = O.fk(ch, g["theta"])
    assert np.array_equal(pos, g["positions"])


def test_params_known_answers():
    ps = P.load_params()
    assert ps.gamma_table("sharp")["C"] == 0.012 and ps.gamma_table("sharp")["N+"] == -0.186
    assert ps.weights.w14_elec == 0.8333333333 and ps.weights.w14_vdw == 0.5
    ch = P.build_chain(["ALA"])
    par = ps.resolve(ch)
    assert par.q[ch.atom_index(0, "N")] == -0.4157
    assert par.R[ch.atom_index(0, "CB")] == 1.9080


def test_sample_sphere_matches_oracle():
    for n in (12, 256, 1024):
        assert np.array_equal(P.generate_samples(n).points, O.sample_sphere(n))


def test_bond_tree_parent_pointers():
    ch = P.build_chain(["SER", "ALA", "GLY", "CYS", "ALA"])
    t = P.build_tree(ch)
    assert t.parent[0] == -1 and (t.parent[1:] >= 0).all()
    ca = ch.atom_index(0, "CA")
    assert t.parent[ca] == ch.atom_index(0, "N")


def test_config_validation_matches_reference():
    with pytest.raises(P.ConfigurationError):
        P.StepConfig(kappa=0.0)
    with pytest.raises(P.ConfigurationError):
        P.Cutoffs(elec=-1.0)
    with pytest.raises(P.ConfigurationError):
        P.SolvationConfig(samples=11)
    with pytest.raises(P.ConfigurationError):
        P.DielectricModel(mode="nope")
    with pytest.raises(P.ConfigurationError):
        P.generate_samples(11)


# ---- the C ABI -------------------------------------------------------------------

def _header_functions():
    text = open(os.path.join(ROOT, "include", "kfb200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    declared = _header_functions()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(N.exported_symbols()) == declared


def test_struct_layouts_and_abi_version():
    lib = N.lib()
    assert lib.kf_abi_version() == N.ABI_VERSION
    for k, cls in enumerate((N.KfChain, N.KfField, N.KfStatus, N.KfBatch, N.KfStep)):
        assert lib.kf_struct_size(k) == ctypes.sizeof(cls)


def test_library_is_built_for_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


# ---- API surface and the no-fallback contract -------------------------------------

REFERENCE_NAMES = """Chain Conformation PeptideGeometry apply_deltas build_chain forward_kinematics
kinematic_state link_transforms KinefoldError AtomParams DielectricModel EnergyBreakdown elec_energy
elec_forces vdw_energy vdw_forces dihedral_angle rotation_about_axis Field FieldConfig JointTorques
StepConfig Trajectory fold hinge_scan joint_torques kcm_step link_wrenches ramachandran_scan
single_point ParamSet load_params ResidueSpec default_templates SampleSphere SasaResult
SolvationConfig generate_samples sasa_pass solvation_forces Cutoffs GridConfig HashGrid
NeighborTable build_grid build_neighbor_table filtered_lists filtered_pairs BondTree
InteractionClass TreeWeights UniformWeights WeightTable build_tree classify""".split()


def test_reference_hot_path_names_present():
    """kinefold/__init__.py:13-85 minus out-of-scope I/O (PDB / RunLog / manifests)."""
    missing = [nm for nm in REFERENCE_NAMES if not hasattr(P, nm)]
    assert not missing, missing


@pytest.mark.skipif(have_gpu(), reason="checks the CPU-only behaviour")
def test_hot_path_has_no_cpu_fallback():
    ch, params, w, fld = make_system(["ALA", "ALA"])
    with pytest.raises(P.NativeLibraryError):
        P.forward_kinematics(ch, ch.conf_zp())
    with pytest.raises(P.NativeLibraryError):
        fld.evaluate(np.zeros((ch.n_atoms, 3)) + np.arange(ch.n_atoms)[:, None])
    with pytest.raises(P.NativeLibraryError):
        P.fold(ch, ch.conf_zp(), fld, P.StepConfig(max_iters=2))


@pytest.mark.parametrize("n", [12, 100, 1024, 4096])
def test_sample_groups_partition_and_cones(n):
    """Hot-path sample groups (solvation.sample_groups): every sample in exactly
    one group of <= 32, and each group's cone bounds all its members."""
    from paper_1712_05012_b200 import solvation as S
    pts = np.asarray(S.generate_samples(n).points)
    groups, cones = S.sample_groups(pts)
    assert np.array_equal(np.sort(np.concatenate(groups)), np.arange(n))
    assert all(0 < len(ix) <= 32 for ix in groups)
    for g, ix in enumerate(groups):
        assert cones[g, 5] == len(ix)
        assert np.all(pts[ix] @ cones[g, :3].astype(float) >= cones[g, 3] - 1e-6)
        assert abs(cones[g, 3] ** 2 + cones[g, 4] ** 2 - 1.0) < 1e-5


@pytest.mark.parametrize("seq", [["ALA", "CYS", "SER"] * 12, (["GLY", "ALA"] * 9) + ["SER"]])
def test_class_codes_match_tree_classes(seq):
    """The cluster kernel's host-built class tables (device.class_codes per (quad,
    window octet) and device.unit_codes per (unit, lane)) against the bond tree's
    classes as the oracle restates them (topology.py:153-195), pair by pair: the 2-bit
    code of lane l is 4 - class(i, j) with i = 4Q + l % 4, j = 8(Q // 2 + k) + l // 4,
    the unit words regroup quads 2U and 2U + 1, and their window bits flag the
    octets holding a class < 4 pair."""
    from paper_1712_05012_b200 import device as DV
    ch = P.build_chain(seq)
    tree = P.build_tree(ch)
    n = ch.n_atoms
    codes = DV.class_codes(tree)
    _, slow = DV.class_window(tree)
    units = DV.unit_codes(codes, slow)
    nq, no = (n + 3) // 4, (n + 7) // 8
    assert codes.shape == (nq, 5) and units.shape == (no, 32)
    for Q in range(nq):
        for k in range(5):
            for lane in range(32):
                i, j = 4 * Q + lane % 4, 8 * (Q // 2 + k) + lane // 4
                want = 0 if (i >= n or j >= n or i == j) else 4 - int(O.classes(tree, np.array([i]), np.array([j]))[0])
                got = (int(codes[Q, k]) >> (2 * lane)) & 3
                assert got == want, (Q, k, lane, got, want)
                U, half = divmod(Q, 2)
                assert (int(units[U, lane]) >> (10 * half + 2 * k)) & 3 == want
    for U in range(no):
        for half in range(2):
            Q = 2 * U + half
            win = [(Q < nq and codes[Q, k] != 0) for k in range(5)]
            assert all(((int(units[U, 0]) >> (20 + 5 * half + k)) & 1) == w for k, w in enumerate(win))
        assert ((int(units[U, 0]) >> 30) & 1) == bool(slow[8 * U:8 * U + 8].any())
