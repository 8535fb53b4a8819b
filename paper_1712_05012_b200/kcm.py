"""Kinetostatic compliance: field evaluation, torques, the step and the loop.

Drop-in mirror of /root/reference/pkg/src/kinefold/kcm.py.  Every numeric
step runs on the GPU:

* ``Field.evaluate`` (kcm.py:104-150): hash-grid binning + fused pair kernel
  (+ fused solvation kernel) + deterministic energy reduction;
* ``link_wrenches`` / ``joint_torques`` (kcm.py:177-240): wrench kernel +
  one-CTA suffix scan;
* ``kcm_step`` (kcm.py:264-274): max-reduction + normalised step;
* ``fold`` (kcm.py:302-351): the whole iteration body replayed from a CUDA
  graph with device-side records and stop tests (``kf_fold_iterations``),
  polled by the host once per chunk.

``fold_ensemble`` is the batched form (one chain, B independent
trajectories; §8(e) of SURVEY.md) that ``paper_1712_05012_b200.ensemble``
shards across GPUs.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from .chain import Conformation, kinematic_state
from .errors import ConfigurationError
from .forcefield import DielectricModel, EnergyBreakdown
from .solvation import SampleSphere, SolvationConfig, generate_samples
from .spatial import Cutoffs, GridConfig


@dataclass(frozen=True)
class FieldConfig:
    solvation: bool = False
    dielectric: DielectricModel = field(default_factory=DielectricModel)
    grid: GridConfig = field(default_factory=GridConfig)
    solvation_cfg: SolvationConfig = field(default_factory=SolvationConfig)
    use_hash: bool = True

    @property
    def cutoffs(self) -> Cutoffs:
        return self.grid.cutoffs

    def active_cutoff(self) -> float:
        c = self.cutoffs
        return max(c.elec, c.vdw, c.cav) if self.solvation else max(c.elec, c.vdw)


@dataclass
class FieldResult:
    forces: np.ndarray
    energy: EnergyBreakdown
    timings: dict
    sasa: object = None


@dataclass
class Field:
    """Parameters, pair weights and options of one system (kcm.py:79-150)."""

    params: object
    weights: object
    config: FieldConfig = field(default_factory=FieldConfig)
    _sphere: SampleSphere | None = None

    def sphere(self) -> SampleSphere:
        cfg = self.config.solvation_cfg
        if self._sphere is None or self._sphere.n != cfg.samples:
            self._sphere = generate_samples(cfg.samples, cfg.sampling, cfg.seed)
        return self._sphere

    def evaluate(self, positions, *, energy_only: bool = False) -> FieldResult:
        from . import device
        return device.evaluate(self, positions, energy_only=energy_only)


@dataclass
class LinkWrenches:
    force: np.ndarray
    torque: np.ndarray


def link_wrenches(chain, positions, forces) -> LinkWrenches:
    from . import device
    f, t = device.link_wrenches(chain, positions, forces)
    return LinkWrenches(force=f, torque=t)


@dataclass
class JointTorques:
    tau: np.ndarray


def joint_torques(chain, conf: Conformation, wrenches: LinkWrenches, state=None) -> JointTorques:
    from . import device
    if state is None:
        state = kinematic_state(chain, conf)
    return JointTorques(tau=device.joint_torques(chain, state, wrenches))


@dataclass(frozen=True)
class StepConfig:
    kappa: float = 0.5
    max_iters: int = 2000
    torque_tol: float = 0.0
    torque_tol_rel: float = 1e-4
    energy_window: int = 20
    energy_tol: float = 0.02
    snapshot_every: int = 50

    def __post_init__(self):
        if self.kappa <= 0:
            raise ConfigurationError("kappa must be positive")
        if min(self.torque_tol, self.torque_tol_rel, self.energy_tol) < 0:
            raise ConfigurationError("tolerances must be non-negative")


def kcm_step(torques: JointTorques, conf: Conformation, config: StepConfig):
    """Normalised compliance step on the GPU (kcm.py:264-274, chain.py:93-101)."""
    from . import device
    if not (~conf.frozen).any():
        raise ConfigurationError("cannot step with every joint frozen")
    theta, deltas, moved = device.kcm_step(np.asarray(torques.tau, float), conf, config.kappa)
    if not moved:
        return conf, np.zeros_like(np.asarray(torques.tau, float))
    return replace(conf, theta=theta), deltas


@dataclass
class IterationRecord:
    index: int
    energy: EnergyBreakdown
    tau_max: float
    timings: dict
    theta: np.ndarray


@dataclass
class Trajectory:
    records: list
    snapshots: list
    final: Conformation
    converged: bool
    reason: str

    @property
    def iterations(self) -> int:
        return len(self.records)

    def energies(self) -> np.ndarray:
        return np.array([r.energy.g_total for r in self.records])


def fold(chain, conf: Conformation, fld: Field, step: StepConfig = StepConfig()) -> Trajectory:
    """KCM loop on the GPU (kcm.py:302-351): identical records, stop rules,
    snapshots and error messages ("aborted at iteration {it}: ...")."""
    from . import device
    return device.fold(chain, conf, fld, step)


def fold_ensemble(chain, confs, fld: Field, step: StepConfig = StepConfig(), *,
                  record_theta: bool = False):
    """B independent trajectories of one chain in one batched launch sequence.

    Returns ``device.EnsembleResult`` (final theta [B, D], per-iteration
    energies and tau_max [B, K, 4], iterations, reasons).  Semantics per
    trajectory are those of ``fold``; an error in any trajectory aborts the
    batch like the reference CLI's ``--batch`` (cli.py:343-347).
    """
    from . import device
    return device.fold_ensemble(chain, confs, fld, step, record_theta=record_theta)


# --------------------------------------------------------------------------
# energy-only scans (kcm.py:358-419): batched single points on the GPU
# --------------------------------------------------------------------------

def single_point(chain, conf: Conformation, fld: Field) -> EnergyBreakdown:
    from . import device
    return device.single_points(chain, [conf.theta], fld)[0]


@dataclass
class ScanGrid:
    axes: list
    dofs: list
    g_elec: np.ndarray
    g_vdw: np.ndarray
    g_cav: np.ndarray

    @property
    def g_total(self) -> np.ndarray:
        return self.g_elec + self.g_vdw + self.g_cav


def ramachandran_scan(chain, residue: int, resolution: int, fld: Field,
                      base: Conformation | None = None) -> ScanGrid:
    if resolution < 2:
        raise ConfigurationError("grid resolution must be at least 2")
    base = base or chain.conf_zp()
    phis = np.linspace(-180.0, 180.0, resolution, endpoint=False)
    psis = np.linspace(-180.0, 180.0, resolution, endpoint=False)
    return _sweep(chain, fld, base, [chain.dof_phi(residue), chain.dof_psi(residue)],
                  [phis + 180.0, psis + 180.0], [phis, psis])


def hinge_scan(chain, hinge_dofs: list, half_range: float, steps: int, fld: Field,
               base: Conformation) -> ScanGrid:
    for dof in hinge_dofs:
        if not 0 <= dof < chain.n_dof:
            raise ConfigurationError(f"hinge joint {dof} out of range")
    if not 1 <= len(hinge_dofs) <= 2:
        raise ConfigurationError("hinge scans support one or two joints")
    if steps < 1:
        raise ConfigurationError("steps must be positive")
    offsets = np.linspace(-half_range, half_range, steps) if steps > 1 else np.zeros(1)
    return _sweep(chain, fld, base, list(hinge_dofs),
                  [base.theta[d] + offsets for d in hinge_dofs], [offsets for _ in hinge_dofs])


def _sweep(chain, fld, base, dofs, theta_axes, label_axes) -> ScanGrid:
    """All grid points as one batch (B = grid size) of FK + field evaluations."""
    from . import device
    shape = tuple(len(a) for a in theta_axes)
    thetas = []
    for idx in np.ndindex(*shape):
        theta = base.theta.copy()
        for d, ax, k in zip(dofs, theta_axes, idx):
            theta[d] = ax[k]
        thetas.append(replace(base, theta=theta).theta)
    energies = device.single_points(chain, thetas, fld)
    g = np.array([[e.g_elec, e.g_vdw, e.g_cav] for e in energies]).reshape(shape + (3,))
    return ScanGrid(axes=list(label_axes), dofs=list(dofs),
                    g_elec=g[..., 0].copy(), g_vdw=g[..., 1].copy(), g_cav=g[..., 2].copy())
