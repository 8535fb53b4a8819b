"""Force-field parameter tables (setup data, off the hot path).

``load_params()`` returns the reference's shipped table
(/root/reference/pkg/src/kinefold/data/params.ff:14-62) held as Python data;
``load_params(path)`` reads a user file in the same sectioned text format
(pdbio.py:196-241).  ``ParamSet.resolve`` maps a chain's atom classes to the
per-atom structure-of-arrays the device tables are built from
(pdbio.py:174-193), including the by-element fallback.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import ParameterFileError
from .forcefield import AtomParams
from .topology import WeightTable

_SHIPPED_WEIGHTS = {"w13_elec": 0.0, "w13_vdw": 0.0,
                    "w14_elec": 0.8333333333, "w14_vdw": 0.5}

_SHIPPED_GAMMA = {
    "sharp": {"C": 0.012, "O/N": -0.116, "S": -0.018, "O-": -0.175,
              "N+": -0.186, "NONE": 0.0},
    "kyte": {"C": 0.004, "O/N": -0.113, "S": -0.017, "O-": -0.166,
             "N+": -0.169, "NONE": 0.0},
}

# class -> (charge e, vdW radius A, well depth kcal/mol, solvation class)
_SHIPPED_CLASSES = {
    "N": (-0.4157, 1.8240, 0.1700, "O/N"),
    "H": (0.2719, 0.6000, 0.0157, "NONE"),
    "C": (0.5973, 1.9080, 0.0860, "C"),
    "O": (-0.5679, 1.6612, 0.2100, "O/N"),
    "O2": (-0.5679, 1.6612, 0.2100, "O-"),
    "CA_GLY": (-0.0252, 1.9080, 0.1094, "C"),
    "CA_ALA": (0.0337, 1.9080, 0.1094, "C"),
    "CA_SER": (-0.0249, 1.9080, 0.1094, "C"),
    "CA_CYS": (0.0213, 1.9080, 0.1094, "C"),
    "HA_GLY": (0.0698, 1.3870, 0.0157, "NONE"),
    "HA_ALA": (0.0823, 1.3870, 0.0157, "NONE"),
    "HA_SER": (0.0843, 1.3870, 0.0157, "NONE"),
    "HA_CYS": (0.1124, 1.3870, 0.0157, "NONE"),
    "CB_ALA": (-0.1825, 1.9080, 0.1094, "C"),
    "HB_ALA": (0.0603, 1.4870, 0.0157, "NONE"),
    "CB_SER": (0.2117, 1.9080, 0.1094, "C"),
    "HB_SER": (0.0352, 1.3870, 0.0157, "NONE"),
    "OG_SER": (-0.6546, 1.7210, 0.2104, "O/N"),
    "HG_SER": (0.4275, 0.3000, 0.0157, "NONE"),
    "CB_CYS": (-0.1231, 1.9080, 0.1094, "C"),
    "HB_CYS": (0.1112, 1.3870, 0.0157, "NONE"),
    "SG_CYS": (-0.3119, 2.0000, 0.2500, "S"),
    "HG_CYS": (0.1933, 0.6000, 0.0157, "NONE"),
}

_ELEMENT_FALLBACK = {
    "C": (0.0, 1.9080, 0.1094, "C"),
    "N": (0.0, 1.8240, 0.1700, "O/N"),
    "O": (0.0, 1.6612, 0.2100, "O/N"),
    "S": (0.0, 2.0000, 0.2500, "S"),
    "H": (0.0, 1.0000, 0.0157, "NONE"),
    "P": (0.0, 2.1000, 0.2000, "NONE"),
}
_GENERIC_FALLBACK = (0.0, 1.5, 0.05, "NONE")


@dataclass
class ParamSet:
    classes: dict
    weights: WeightTable
    gamma_sets: dict

    def gamma_table(self, which: str = "sharp") -> dict:
        if which not in self.gamma_sets:
            raise ParameterFileError(f"no solvation parameter set {which!r}")
        return self.gamma_sets[which]

    def resolve(self, chain, gamma_set: str = "sharp") -> AtomParams:
        gam = self.gamma_table(gamma_set)
        rows = []
        for cls, elem in zip(chain.atom_classes, chain.atom_elements):
            row = self.classes.get(cls)
            if row is None:
                row = _ELEMENT_FALLBACK.get(elem, _GENERIC_FALLBACK)
            if row[3] not in gam:
                raise ParameterFileError(f"solvation class {row[3]!r} missing from table")
            rows.append(row)
        q = np.array([r[0] for r in rows], dtype=float)
        radius = np.array([r[1] for r in rows], dtype=float)
        eps = np.array([r[2] for r in rows], dtype=float)
        gamma = np.array([gam[r[3]] for r in rows], dtype=float)
        return AtomParams(q=q, R=radius, eps=eps, gamma=gamma,
                          solv_class=tuple(r[3] for r in rows))


def load_params(path=None) -> ParamSet:
    if path is None:
        return ParamSet(classes=dict(_SHIPPED_CLASSES),
                        weights=WeightTable(**_SHIPPED_WEIGHTS),
                        gamma_sets={k: dict(v) for k, v in _SHIPPED_GAMMA.items()})
    return _parse(Path(path).read_text(), str(path))


def _parse(text: str, source: str) -> ParamSet:
    classes, gammas, weights = {}, {}, dict(
        w13_elec=0.0, w13_vdw=0.0, w14_elec=1.0 / 1.2, w14_vdw=0.5)
    section = None
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if line.startswith("["):
            section = line.strip("[]").split()
            continue
        tok = line.split()
        where = f"{source}:{lineno}"
        try:
            if section == ["weights"]:
                if tok[0] not in weights:
                    raise ParameterFileError(f"{where}: unknown weight {tok[0]!r}")
                weights[tok[0]] = float(tok[1])
            elif section and section[0] == "gamma":
                gammas.setdefault(section[1], {})[tok[0]] = float(tok[1])
            elif section == ["classes"]:
                if len(tok) != 5:
                    raise ParameterFileError(f"{where}: class rows need 5 fields")
                if tok[0] in classes:
                    raise ParameterFileError(f"{where}: duplicate class {tok[0]!r}")
                classes[tok[0]] = (float(tok[1]), float(tok[2]), float(tok[3]), tok[4])
            else:
                raise ParameterFileError(f"{where}: content outside any section")
        except (ValueError, IndexError) as exc:
            raise ParameterFileError(f"{where}: {exc}") from exc
    if not classes:
        raise ParameterFileError(f"{source}: no [classes] section")
    if not gammas:
        raise ParameterFileError(f"{source}: no [gamma] sections")
    return ParamSet(classes=classes, weights=WeightTable(**weights), gamma_sets=gammas)
