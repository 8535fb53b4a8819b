"""Electrostatic and van der Waals terms: types and the drop-in API functions.

Types mirror /root/reference/pkg/src/kinefold/forcefield.py:22-78.  The API
functions (``extract_pairs``, ``elec_energy`` / ``elec_forces`` / ``vdw_energy``
/ ``vdw_forces``, ``elec_pair_quantities`` / ``vdw_pair_quantities``,
``accumulate_pair_forces``; forcefield.py:81-172) run on the GPU through
``kf_filter_table`` / ``kf_compact_pairs`` / ``kf_pair_terms`` with the
reference's fp64 formulas.  Inside the KCM loop the same terms are computed by
the fused pair kernel instead (csrc/kf_nonbonded.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError

COULOMB_K = 332.06
MIN_DISTANCE = 1e-6


@dataclass(frozen=True)
class AtomParams:
    """Per-atom nonbonded parameters, structure of arrays (forcefield.py:26-48)."""

    q: np.ndarray
    R: np.ndarray
    eps: np.ndarray
    gamma: np.ndarray
    solv_class: tuple

    def __post_init__(self):
        n = len(self.q)
        if any(len(getattr(self, k)) != n for k in ("R", "eps", "gamma")):
            raise ConfigurationError("parameter arrays must share one length")
        if np.any(np.asarray(self.R) <= 0):
            raise ConfigurationError("van der Waals radii must be positive")
        if np.any(np.asarray(self.eps) < 0):
            raise ConfigurationError("well depths must be non-negative")

    @property
    def n_atoms(self) -> int:
        return len(self.q)


@dataclass(frozen=True)
class DielectricModel:
    """kappa(d) = d ("distance") or a constant (forcefield.py:51-67)."""

    mode: str = "distance"
    kappa: float = 1.0

    def __post_init__(self):
        if self.mode not in ("distance", "constant"):
            raise ConfigurationError(f"unknown dielectric mode {self.mode!r}")
        if self.kappa <= 0:
            raise ConfigurationError("kappa must be positive")

    def of(self, d) -> np.ndarray:
        if self.mode == "distance":
            return np.asarray(d, float)
        return np.full(np.shape(d), self.kappa)


@dataclass(frozen=True)
class EnergyBreakdown:
    g_elec: float
    g_vdw: float
    g_cav: float

    @property
    def g_total(self) -> float:
        return self.g_elec + self.g_vdw + self.g_cav


def extract_pairs(positions, table, d_cut: float):
    """Cut-off pairs (i < j, d) of a superset table with the clash guard
    (forcefield.py:81-89); filtering and compaction on the GPU."""
    from . import device
    return device.extract_pairs(positions, table, d_cut)


def elec_pair_quantities(params, i, j, d, w, dielectric):
    """Per-pair Coulomb energy and force magnitude (forcefield.py:98-103)."""
    from . import device
    return device.pair_quantities(params, i, j, d, w, 0, dielectric)


def vdw_pair_quantities(params, i, j, d, w):
    """Per-pair 6-12 energy and force magnitude (forcefield.py:106-113)."""
    from . import device
    return device.pair_quantities(params, i, j, d, w, 1, None)


def accumulate_pair_forces(n, positions, i, j, d, mag) -> np.ndarray:
    """Scatter +/- mag * e_ij (forcefield.py:116-117, :162-172)."""
    from . import device
    return device.accumulate_pair_forces(n, positions, i, j, d, mag)


def elec_energy(positions, params: AtomParams, table, weights, d_cut: float = 9.0,
                dielectric: DielectricModel = DielectricModel()) -> float:
    from . import device
    return device.table_term(positions, params, table, weights, d_cut, dielectric, 0, "energy")


def elec_forces(positions, params: AtomParams, table, weights, d_cut: float = 9.0,
                dielectric: DielectricModel = DielectricModel()) -> np.ndarray:
    from . import device
    return device.table_term(positions, params, table, weights, d_cut, dielectric, 0, "forces")


def vdw_energy(positions, params: AtomParams, table, weights, d_cut: float = 5.0) -> float:
    from . import device
    return device.table_term(positions, params, table, weights, d_cut, None, 1, "energy")


def vdw_forces(positions, params: AtomParams, table, weights, d_cut: float = 5.0) -> np.ndarray:
    from . import device
    return device.table_term(positions, params, table, weights, d_cut, None, 1, "forces")
