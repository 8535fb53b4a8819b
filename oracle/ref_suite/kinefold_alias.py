"""pytest plugin (test infrastructure): run the reference package's own test
suite against this package by aliasing ``kinefold`` and its submodules to
``paper_1712_05012_b200`` (SURVEY.md §4's reuse plan).

    python -m pytest -p oracle.ref_suite.kinefold_alias oracle/_ref/pkg_tests ...

Modules of the reference that this package does not rebuild (out of scope per
SURVEY.md §2 / §8: PDB reading, the CLI, the template parser) are provided
only as far as the hot path needs them; the tests that exercise the missing
parts are deselected by name in ``DESELECT`` below, each with its reason.
"""

from __future__ import annotations

import sys
import types

import paper_1712_05012_b200 as P
from paper_1712_05012_b200 import (chain, errors, forcefield, geometry, kcm, params, residues, runlog,
                                   solvation, spatial, topology)

# kinefold.pdbio = the parameter file (ParamSet, load_params) + the run outputs
# (RunLog, write_manifest, write_pdb) of this package; read_pdb and friends are
# the out-of-scope importer.
pdbio = types.ModuleType("kinefold.pdbio")
for _m in (params, runlog):
    for _k in dir(_m):
        if not _k.startswith("__"):
            setattr(pdbio, _k, getattr(_m, _k))


def _out_of_scope(*_a, **_k):
    raise NotImplementedError("PDB reading is out of scope for this package (SURVEY.md §2)")


pdbio.read_pdb = _out_of_scope

ALIASES = {"kinefold": P, "kinefold.chain": chain, "kinefold.errors": errors, "kinefold.forcefield": forcefield,
           "kinefold.geometry": geometry, "kinefold.kcm": kcm, "kinefold.residues": residues,
           "kinefold.solvation": solvation, "kinefold.spatial": spatial, "kinefold.topology": topology,
           "kinefold.pdbio": pdbio}
for _name, _mod in ALIASES.items():
    sys.modules[_name] = _mod

# test id substring -> reason (out of scope, or a deliberate deviation)
DESELECT = {
    "test_cli.py": "the CLI's argument parsing is out of scope (SURVEY.md §2); its fold --batch and bench "
                   "outputs are covered by tests/test_runlog.py against files the reference CLI wrote",
    "test_imported.py": "imported-structure chain building from PDB files is out of scope (SURVEY.md §2)",
    "test_pdbio.py": "PDB reading / the parameter-file error paths are out of scope (SURVEY.md §2)",
    "test_residues.py": "the residue-template parser is out of scope (SURVEY.md §2); the shipped templates "
                        "are restated as data",
    "test_hinge_minimum_near_native_after_reimport": "re-imports a written PDB (read_pdb + imported-structure "
                                                     "building: out of scope)",
    "test_hetero_pairs_classified_full": "builds a hetero chain from a StructureRecord (the out-of-scope PDB "
                                         "importer)",
}

# With the default fp32 pair math (set_pair_precision, KFB200_PAIR_PRECISION) these
# tests ask for more than fp32 rounding gives; they pass in fp64 mode (the suite is
# run in both modes by tests/test_reference_suite.py).
XFAIL_FP32 = {
    "test_torque_is_energy_gradient": "central difference with h = 1e-5 degrees: energy differences of ~1e-8 "
                                      "relative, below the fp32 pair energies' ~1e-7 rounding",
    "test_polyglycine_mirror_symmetry": "mirror energies equal to rel 1e-8; fp32 pair rounding differs ~1e-7 "
                                        "between the two conformations",
    "test_criterion_12_mirror_symmetry": "as test_polyglycine_mirror_symmetry (acceptance criterion 12)",
    "test_solvated_helix_keeps_right_handed_region": "asserts convergence within a fixed iteration budget; the "
                                                     "fp32 trajectory's plateau test fires at another iteration",
}


def pytest_collection_modifyitems(config, items):
    import pytest
    from paper_1712_05012_b200 import pair_precision
    keep, drop = [], []
    for it in items:
        reason = next((r for k, r in DESELECT.items() if k in it.nodeid), None)
        (drop if reason else keep).append(it)
        why = next((r for k, r in XFAIL_FP32.items() if k in it.nodeid), None)
        if why and pair_precision() == "fp32":
            it.add_marker(pytest.mark.xfail(reason="fp32 pair math: " + why, strict=False))
    if drop:
        config.hook.pytest_deselected(items=drop)
        items[:] = keep


def pytest_ignore_collect(collection_path, config):
    # whole modules of out-of-scope subsystems (they import its names at module level)
    return collection_path.name in DESELECT
