"""Kinematic chain model: conformations, link records, forward kinematics.

Types and the canonical builder mirror /root/reference/pkg/src/kinefold/
chain.py (``Conformation`` :73-90, ``LinkRecord`` :104-116, ``Chain`` :119-223,
``build_chain`` :394-525).  Chain construction is once-per-system host setup;
``kinematic_state`` / ``forward_kinematics`` (chain.py:240-276) run the FK
kernel (csrc/kf_kinematics.cu) through the C-ABI and have no CPU fallback.

Functions accept any duck-typed chain with the reference's attributes, so a
``kinefold.Chain`` built by the reference works unchanged.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

from .errors import ChainBuildError, ConfigurationError, UnknownResidueError
from .geometry import (dihedral_angle, frame_from_backbone, signed_degrees,
                       unit_vector, wrap_degrees)
from .residues import default_templates

# canonical backbone constants (chain.py:39-57)
BOND_N_CA, BOND_CA_C, BOND_C_N = 1.47, 1.53, 1.32
ANGLE_N_CA_C, ANGLE_CA_C_N, ANGLE_C_N_CA = 111.0, 114.5, 123.0
BOND_C_O_TERM, ANGLE_CA_C_O_TERM = 1.25, 117.0
BOND_N_H_TERM, ANGLE_H_N_CA = 1.01, 119.0
PLANE_CONSTANTS = {
    "CA_C": (-0.2761, 1.4488),
    "C_N": (1.2761, -1.4488),
    "C_O": (-1.3324, 2.3401),
    "N_H": (1.4103, -2.5111),
}
MAX_LINKS_PER_RESIDUE = 6


@dataclass(frozen=True)
class PeptideGeometry:
    plane_constants: dict = field(default_factory=lambda: dict(PLANE_CONSTANTS))
    omega_mode: str = "trans"


@dataclass(frozen=True)
class Conformation:
    """theta per joint (degrees, wrapped into [0, 360)) plus a frozen mask."""

    theta: np.ndarray
    frozen: np.ndarray
    residue_count: int

    def __post_init__(self):
        object.__setattr__(self, "theta", wrap_degrees(np.asarray(self.theta, float)))
        object.__setattr__(self, "frozen", np.asarray(self.frozen, bool).copy())
        if self.theta.shape != self.frozen.shape:
            raise ConfigurationError("theta and frozen mask must have equal length")

    def freeze(self, dofs) -> "Conformation":
        mask = self.frozen.copy()
        mask[np.asarray(dofs, int)] = True
        return replace(self, frozen=mask)


def apply_deltas(conf: Conformation, deltas) -> Conformation:
    """theta + delta on free joints, wrapped (chain.py:93-101)."""
    deltas = np.asarray(deltas, float)
    if deltas.shape != conf.theta.shape:
        raise ConfigurationError(
            f"delta length {deltas.shape} != dof count {conf.theta.shape}")
    step = np.where(conf.frozen, 0.0, deltas)
    return replace(conf, theta=wrap_degrees(conf.theta + step))


@dataclass(frozen=True)
class LinkRecord:
    index: int
    kind: str
    residue: int
    chi_index: int
    dof: int
    parent: int
    axis0: np.ndarray | None
    body0: np.ndarray
    point0: np.ndarray
    atom_indices: np.ndarray
    chi0: float = 0.0


@dataclass
class Chain:
    residues: list
    links: list
    atom_names: list
    atom_elements: list
    atom_classes: list
    atom_residue: np.ndarray
    atom_link: np.ndarray
    zp_pos: np.ndarray
    bonds: list
    hetero_mask: np.ndarray
    geometry: PeptideGeometry
    source: str = "canonical"

    def __post_init__(self):
        self._lookup = {}
        for k, (r, nm) in enumerate(zip(self.atom_residue, self.atom_names)):
            self._lookup.setdefault((int(r), nm), k)

    n_atoms = property(lambda self: len(self.atom_names))
    n_residues = property(lambda self: len(self.residues))
    n_dof = property(lambda self: len(self.links) - 1)

    def atom_index(self, residue: int, name: str) -> int:
        return self._lookup[(residue, name)]

    def dof_phi(self, i: int) -> int:
        return 2 * i

    def dof_psi(self, i: int) -> int:
        return 2 * i + 1

    def dof_chi(self, i: int, k: int) -> int:
        return self.links[self._chi_link_index(i, k)].dof

    def side_dofs(self, i: int) -> list:
        return [l.dof for l in self.links if l.kind == "chi" and l.residue == i]

    def _chi_link_index(self, i: int, k: int) -> int:
        for li, l in enumerate(self.links):
            if l.kind == "chi" and l.residue == i and l.chi_index == k:
                return li
        raise KeyError(f"residue {i} has no chi joint {k}")

    def conf_zp(self) -> Conformation:
        return Conformation(np.zeros(self.n_dof), np.zeros(self.n_dof, bool),
                            self.n_residues)

    def conf_from_backbone(self, phi, psi) -> Conformation:
        m = self.n_residues
        theta = np.zeros(self.n_dof)
        theta[0:2 * m:2] = wrap_degrees(np.broadcast_to(np.asarray(phi, float), (m,)) + 180.0)
        theta[1:2 * m:2] = wrap_degrees(np.broadcast_to(np.asarray(psi, float), (m,)) + 180.0)
        return Conformation(theta, np.zeros(self.n_dof, bool), m)

    def dihedrals_from_theta(self, conf: Conformation):
        m = self.n_residues
        phi = signed_degrees(conf.theta[0:2 * m:2] - 180.0)
        psi = signed_degrees(conf.theta[1:2 * m:2] - 180.0)
        chi = {(l.residue, l.chi_index): float(signed_degrees(conf.theta[l.dof] + l.chi0))
               for l in self.links if l.kind == "chi"}
        return phi, psi, chi

    def theta_from_dihedrals(self, phi, psi, chi=None) -> Conformation:
        conf = self.conf_from_backbone(phi, psi)
        if chi:
            theta = conf.theta.copy()
            for (i, k), value in chi.items():
                link = self.links[self._chi_link_index(i, k)]
                theta[link.dof] = wrap_degrees(value - link.chi0)
            conf = replace(conf, theta=theta)
        return conf

    def validate_conformation(self, conf: Conformation) -> None:
        if conf.theta.shape[0] != self.n_dof:
            raise ConfigurationError(
                f"conformation has {conf.theta.shape[0]} dofs, chain needs {self.n_dof}")


# --------------------------------------------------------------------------
# forward kinematics (device)
# --------------------------------------------------------------------------

@dataclass
class KinematicState:
    """Per-link rotation M, joint point P, current axis U (None for ground),
    and atom positions (chain.py:230-237)."""

    transforms: list
    joint_points: list
    axes: list
    positions: np.ndarray


def kinematic_state(chain, conf: Conformation) -> KinematicState:
    """Prefix composition of link transforms on the GPU (chain.py:240-261)."""
    from . import device
    _validate(chain, conf)
    M, P, U, pos = device.kinematic_state(chain, conf.theta)
    axes = [None if l.kind == "ground" else U[li] for li, l in enumerate(chain.links)]
    return KinematicState(transforms=list(M), joint_points=list(P), axes=axes,
                          positions=pos)


def forward_kinematics(chain, conf: Conformation) -> np.ndarray:
    from . import device
    _validate(chain, conf)
    return device.kinematic_state(chain, conf.theta, positions_only=True)


def measure_backbone_dihedrals(chain: Chain, positions: np.ndarray):
    """(phi, psi) of every residue measured from coordinates, NaN where the
    neighbouring residue is missing (chain.py:279-294 of the reference: phi from
    C(i-1), N, CA, C; psi from N, CA, C, N(i+1)).  Host geometry, not on the
    iteration's path."""
    m = chain.n_residues
    pos = np.asarray(positions, float)
    phi = np.full(m, np.nan)
    psi = np.full(m, np.nan)
    for r in range(m):
        n_r, ca_r, c_r = (pos[chain.atom_index(r, a)] for a in ("N", "CA", "C"))
        if r > 0:
            phi[r] = dihedral_angle(pos[chain.atom_index(r - 1, "C")], n_r, ca_r, c_r)
        if r + 1 < m:
            psi[r] = dihedral_angle(n_r, ca_r, c_r, pos[chain.atom_index(r + 1, "N")])
    return phi, psi


def link_transforms(chain, conf: Conformation) -> list:
    state = kinematic_state(chain, conf)
    out = [None] * (len(chain.links) - 1)
    for li, link in enumerate(chain.links):
        if link.kind != "ground":
            out[link.dof] = state.transforms[li]
    return out


def _validate(chain, conf) -> None:
    if np.asarray(conf.theta).shape[0] != len(chain.links) - 1:
        raise ConfigurationError(
            f"conformation has {np.asarray(conf.theta).shape[0]} dofs, "
            f"chain needs {len(chain.links) - 1}")


# --------------------------------------------------------------------------
# canonical builder (host setup; chain.py:301-555)
# --------------------------------------------------------------------------

def _heading(angle_deg: float) -> np.ndarray:
    a = math.radians(angle_deg)
    return np.array([math.cos(a), math.sin(a), 0.0])


def _planar_backbone(m: int, omegas: list):
    """Zig-zag walk of N, CA and provisional C in the z=0 plane (chain.py:306-326)."""
    n_at, ca_at, c_at = [np.zeros(3)], [], []
    heading, sign = 0.0, 1.0
    for i in range(m):
        ca_at.append(n_at[i] + BOND_N_CA * _heading(heading))
        heading += sign * (180.0 - ANGLE_N_CA_C)
        sign = -sign
        c_at.append(ca_at[i] + BOND_CA_C * _heading(heading))
        if i + 1 == m:
            break
        heading += sign * (180.0 - ANGLE_CA_C_N)
        sign = -sign
        n_at.append(c_at[i] + BOND_C_N * _heading(heading))
        if omegas[i] == "cis":
            sign = -sign
        heading += sign * (180.0 - ANGLE_C_N_CA)
        sign = -sign
    return n_at, ca_at, c_at, heading, sign


def _plane_row(key, b2, b3):
    c1, c2 = PLANE_CONSTANTS[key]
    return c1 * b2 + c2 * b3


class _Assembly:
    def __init__(self):
        self.atoms = []      # (name, element, class, residue, link, xyz)
        self.links = []      # dicts, LinkRecord fields
        self.bonds = []

    def atom(self, name, element, cls, residue, link, xyz) -> int:
        self.atoms.append((name, element, cls, residue, link, np.asarray(xyz, float)))
        return len(self.atoms) - 1

    def link(self, **kw) -> int:
        kw["index"] = len(self.links)
        self.links.append(kw)
        return kw["index"]


def build_chain(sequence, geometry=None, *, omega="trans", templates=None) -> Chain:
    """Canonical extended build from residue codes (chain.py:394-525).

    Imported geometry (``geometry`` not None) is outside this package's scope:
    build such chains with the reference and pass them in (duck-typed).
    """
    if geometry is not None:
        raise ChainBuildError("imported geometry: build the chain with the reference "
                              "package and pass it to this package's hot-path API")
    seq = [str(c).upper() for c in sequence]
    if not seq:
        raise ChainBuildError("zero-length sequence")
    templates = templates or default_templates()
    for code in seq:
        if code not in templates:
            raise UnknownResidueError(f"no residue template for {code!r}")
    m = len(seq)
    omegas = [omega] * max(m - 1, 1) if isinstance(omega, str) else list(omega)
    if len(omegas) != max(m - 1, 1):
        raise ChainBuildError("omega list must have one entry per peptide bond")
    if any(w not in ("trans", "cis") for w in omegas):
        raise ChainBuildError("omega must be trans or cis")

    n_at, ca_at, c_tmp, heading, sign = _planar_backbone(m, omegas)
    c_at, o_at, h_at = [], [], [None] * m
    for i in range(m - 1):
        if omegas[i] == "trans":
            b2 = n_at[i + 1] - ca_at[i]
            b3 = ca_at[i + 1] - n_at[i + 1]
            c = ca_at[i] + _plane_row("CA_C", b2, b3)
            o = c + _plane_row("C_O", b2, b3)
            h_at[i + 1] = n_at[i + 1] + _plane_row("N_H", b2, b3)
        else:
            c = c_tmp[i]
            o = c + BOND_C_O_TERM * unit_vector(
                -(unit_vector(ca_at[i] - c) + unit_vector(n_at[i + 1] - c)))
            h_at[i + 1] = n_at[i + 1] + BOND_N_H_TERM * unit_vector(
                -(unit_vector(c - n_at[i + 1]) + unit_vector(ca_at[i + 1] - n_at[i + 1])))
        c_at.append(c)
        o_at.append(o)
    split = 180.0 - ANGLE_CA_C_O_TERM
    c_last = c_tmp[m - 1]
    oxt = c_last + BOND_C_O_TERM * _heading(heading + sign * split)
    c_at.append(c_last)
    o_at.append(c_last + BOND_C_O_TERM * _heading(heading - sign * split))
    h_at[0] = n_at[0] + BOND_N_H_TERM * _heading(-ANGLE_H_N_CA)

    asm = _Assembly()
    ground = asm.link(kind="ground", residue=-1, chi_index=0, dof=-1, parent=-1,
                      axis0=None, body0=np.zeros(3), point0=np.zeros(3))
    phi_link, psi_link = [], []
    for i in range(m):
        phi_link.append(asm.link(
            kind="phi", residue=i, chi_index=0, dof=2 * i,
            parent=psi_link[i - 1] if i else ground,
            axis0=unit_vector(ca_at[i] - n_at[i]), body0=ca_at[i] - n_at[i],
            point0=n_at[i].copy()))
        tip = n_at[i + 1] if i + 1 < m else oxt
        psi_link.append(asm.link(
            kind="psi", residue=i, chi_index=0, dof=2 * i + 1, parent=phi_link[i],
            axis0=unit_vector(c_at[i] - ca_at[i]), body0=tip - ca_at[i],
            point0=ca_at[i].copy()))

    n_idx, c_idx = [], []
    for i in range(m):
        spec = templates.get(seq[i])
        n_owner = ground if i == 0 else psi_link[i - 1]
        n_idx.append(asm.atom("N", "N", "N", i, n_owner, n_at[i]))
        asm.atom("H", "H", "H", i, n_owner, h_at[i])
        ca = asm.atom("CA", "C", f"CA_{seq[i]}", i, phi_link[i], ca_at[i])
        asm.bonds += [(n_idx[i], ca), (n_idx[i], n_idx[i] + 1)]
        frame = frame_from_backbone(n_at[i], ca_at[i], c_at[i])
        named = {"N": n_idx[i], "CA": ca}
        side = {}
        parent_link = phi_link[i]
        for k in range(1, spec.side_links + 1):
            parent_link = side[k] = asm.link(
                kind="chi", residue=i, chi_index=k, dof=-2, parent=parent_link,
                axis0=None, body0=np.zeros(3), point0=np.zeros(3))
        for ta in spec.atoms:
            owner = phi_link[i] if ta.link == 0 else side[ta.link]
            named[ta.name] = asm.atom(ta.name, ta.element, ta.param_class, i, owner,
                                      ca_at[i] + frame @ ta.local)
        c_idx.append(asm.atom("C", "C", "C", i, psi_link[i], c_at[i]))
        named["C"] = c_idx[i]
        asm.bonds += [(named[ta.parent], named[ta.name]) for ta in spec.atoms]
        o = asm.atom("O", "O", "O", i, psi_link[i], o_at[i])
        asm.bonds += [(ca, c_idx[i]), (c_idx[i], o)]
        if i + 1 == m:
            asm.bonds.append((c_idx[i], asm.atom("OXT", "O", "O2", i, psi_link[i], oxt)))
        for k in range(1, spec.side_links + 1):
            src, dst = spec.joints[k - 1]
            p_src, p_dst = asm.atoms[named[src]][5], asm.atoms[named[dst]][5]
            rec = asm.links[side[k]]
            rec.update(axis0=unit_vector(p_dst - p_src), point0=p_src.copy(),
                       body0=p_dst - p_src)
            if spec.chi_refs and len(spec.chi_refs[k - 1]) == 4:
                rec["chi0"] = dihedral_angle(*[asm.atoms[named[nm]][5]
                                               for nm in spec.chi_refs[k - 1]])
            else:
                rec["chi0"] = (float(spec.rotamer_defaults[k - 1])
                               if spec.rotamer_defaults else 0.0)
    asm.bonds += [(c_idx[i], n_idx[i + 1]) for i in range(m - 1)]
    return _finish(asm, seq, PeptideGeometry(omega_mode=omegas[0]))


def _finish(asm: _Assembly, residues, geometry) -> Chain:
    next_dof = 2 * len(residues)
    for rec in asm.links:
        if rec["kind"] == "chi":
            rec["dof"] = next_dof
            next_dof += 1
    atom_link = np.asarray([a[4] for a in asm.atoms], int)
    links = [LinkRecord(atom_indices=np.flatnonzero(atom_link == rec["index"]), **rec)
             for rec in asm.links]
    chain = Chain(
        residues=list(residues), links=links,
        atom_names=[a[0] for a in asm.atoms], atom_elements=[a[1] for a in asm.atoms],
        atom_classes=[a[2] for a in asm.atoms],
        atom_residue=np.asarray([a[3] for a in asm.atoms], int), atom_link=atom_link,
        zp_pos=np.array([a[5] for a in asm.atoms]), bonds=asm.bonds,
        hetero_mask=np.zeros(len(asm.atoms), bool), geometry=geometry)
    if chain.n_dof > MAX_LINKS_PER_RESIDUE * chain.n_residues:
        raise ChainBuildError("link count exceeds 6 per residue")
    return chain
