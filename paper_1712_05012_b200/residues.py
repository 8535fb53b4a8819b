"""Residue templates (setup data, off the hot path).

The canonical builder needs the side-chain geometry of the residues the
reference ships (GLY, ALA, SER, CYS: /root/reference/pkg/src/kinefold/data/
templates.kft:19-63).  They are held here as Python data rather than a text
file; the numbers are the reference's so built chains are bit-identical.
Local frame: origin CA, x along N->CA, y toward C, z = x cross y
(residues.py:1-7).  ``link`` 0 rides the CA link, k>0 the k-th chi link.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import UnknownResidueError

ONE_TO_THREE = {
    "A": "ALA", "R": "ARG", "N": "ASN", "D": "ASP", "C": "CYS",
    "Q": "GLN", "E": "GLU", "G": "GLY", "H": "HIS", "I": "ILE",
    "L": "LEU", "K": "LYS", "M": "MET", "F": "PHE", "P": "PRO",
    "S": "SER", "T": "THR", "W": "TRP", "Y": "TYR", "V": "VAL",
}


@dataclass(frozen=True)
class TemplateAtom:
    name: str
    element: str
    param_class: str
    parent: str
    link: int
    local: np.ndarray


@dataclass(frozen=True)
class ResidueSpec:
    """One residue type: atoms hanging off CA plus its chi joints."""

    aa_type: str
    side_links: int
    atoms: tuple
    joints: tuple
    chi_refs: tuple = ()
    rotamer_defaults: tuple = ()

    def atom(self, name: str) -> TemplateAtom:
        for a in self.atoms:
            if a.name == name:
                return a
        raise KeyError(name)


@dataclass
class TemplateRegistry:
    specs: dict = field(default_factory=dict)

    def __contains__(self, code) -> bool:
        return code in self.specs

    def get(self, code: str) -> ResidueSpec:
        if code not in self.specs:
            raise UnknownResidueError(f"no residue template for {code!r}")
        return self.specs[code]


# (name, element, class, parent, link, x, y, z) rows per residue type
_HA = (0.347318, -0.497454, 0.905544)
_CB = (0.533315, -0.769587, -1.210046)
_HB_A = (0.178624, -1.799538, -1.171382)
_HB_B = (1.623181, -0.760399, -1.195599)

_TABLE = {
    "GLY": dict(
        atoms=[("HA2", "H", "HA_GLY", "CA", 0, (0.363849, -0.513740, -0.889823)),
               ("HA3", "H", "HA_GLY", "CA", 0, (0.363849, -0.513740, 0.889823))],
        joints=[], chi_refs=[], rotamers=[]),
    "ALA": dict(
        atoms=[("HA", "H", "HA_ALA", "CA", 0, _HA),
               ("CB", "C", "CB_ALA", "CA", 1, _CB),
               ("HB1", "H", "HB_ALA", "CB", 1, _HB_A),
               ("HB2", "H", "HB_ALA", "CB", 1, _HB_B),
               ("HB3", "H", "HB_ALA", "CB", 1, (0.178624, -0.297871, -2.126440))],
        joints=[("CA", "CB")], chi_refs=[("N", "CA", "CB", "HB1")], rotamers=[-60.0]),
    "SER": dict(
        atoms=[("HA", "H", "HA_SER", "CA", 0, _HA),
               ("CB", "C", "CB_SER", "CA", 1, _CB),
               ("HB2", "H", "HB_SER", "CB", 1, _HB_A),
               ("HB3", "H", "HB_SER", "CB", 1, _HB_B),
               ("OG", "O", "OG_SER", "CB", 1, (0.090128, -0.181514, -2.412483)),
               ("HG", "H", "HG_SER", "OG", 2, (0.442543, -0.688553, -3.147544))],
        joints=[("CA", "CB"), ("CB", "OG")],
        chi_refs=[("N", "CA", "CB", "OG"), ("CA", "CB", "OG", "HG")],
        rotamers=[60.0, 180.0]),
    "CYS": dict(
        atoms=[("HA", "H", "HA_CYS", "CA", 0, _HA),
               ("CB", "C", "CB_CYS", "CA", 1, _CB),
               ("HB2", "H", "HB_CYS", "CB", 1, _HB_A),
               ("HB3", "H", "HB_CYS", "CB", 1, _HB_B),
               ("SG", "S", "SG_CYS", "CB", 1, (-0.069384, 0.033152, -2.716188)),
               ("HG", "H", "HG_CYS", "SG", 2, (0.523443, -0.810900, -3.571601))],
        joints=[("CA", "CB"), ("CB", "SG")],
        chi_refs=[("N", "CA", "CB", "SG"), ("CA", "CB", "SG", "HG")],
        rotamers=[60.0, 180.0]),
}


def _make_spec(code: str, row: dict) -> ResidueSpec:
    atoms = tuple(TemplateAtom(n, e, c, p, k, np.array([float(v) for v in xyz]))
                  for n, e, c, p, k, xyz in row["atoms"])
    return ResidueSpec(aa_type=code, side_links=len(row["joints"]), atoms=atoms,
                       joints=tuple(row["joints"]), chi_refs=tuple(row["chi_refs"]),
                       rotamer_defaults=tuple(row["rotamers"]))


_default: TemplateRegistry | None = None


def default_templates() -> TemplateRegistry:
    global _default
    if _default is None:
        _default = TemplateRegistry({c: _make_spec(c, r) for c, r in _TABLE.items()})
    return _default
