"""Cavity (SASA) solvation by sample enumeration: types and the drop-in API.

Types and setup mirror /root/reference/pkg/src/kinefold/solvation.py:32-126
(``SolvationConfig``, the deterministic geodesic ``generate_samples``,
``ExposureStates``, ``SasaResult``, ``check_cav_cutoff``) and the fixed-point
quantum (:184-191).  ``sasa_pass`` (:135-181) and ``solvation_forces``
(:194-255) run on the GPU (csrc/kf_solvation.cu) and are bit-identical to the
reference: same fp64 coverage tests, same int64 fixed point.  ``threads`` is
accepted for API compatibility; the GPU result is schedule-independent like
the reference's.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError

MIN_SAMPLES = 12
FIXED_POINT_BITS = 36


@dataclass(frozen=True)
class SolvationConfig:
    probe_radius: float = 1.4
    delta_r: float = 1e-2
    samples: int = 1024
    sampling: str = "geodesic"
    seed: int = 0
    threads: int = 1

    def __post_init__(self):
        if min(self.probe_radius, self.delta_r) <= 0 or self.samples < MIN_SAMPLES:
            raise ConfigurationError(
                "probe radius and delta_r must be positive, samples >= 12")


@dataclass(frozen=True)
class SampleSphere:
    points: np.ndarray
    mode: str = "geodesic"

    @property
    def n(self) -> int:
        return len(self.points)


def generate_samples(n: int, mode: str = "geodesic", seed: int = 0) -> SampleSphere:
    """Latitude orbits, points per orbit proportional to sin(polar), golden-ratio
    azimuth offsets (solvation.py:64-97).  Once per system, host numpy."""
    if n < MIN_SAMPLES:
        raise ConfigurationError(f"need at least {MIN_SAMPLES} sample points, got {n}")
    if mode == "random":
        v = np.random.default_rng(seed).normal(size=(n, 3))
        return SampleSphere(v / np.linalg.norm(v, axis=1, keepdims=True), mode)
    if mode != "geodesic":
        raise ConfigurationError(f"unknown sampling mode {mode!r}")
    n_orb = max(2 * int(round(math.sqrt(math.pi * n) / 4.0)), 2)
    polar = (np.arange(n_orb) + 0.5) * math.pi / n_orb
    w = np.sin(polar)
    ideal = n * w / w.sum()
    per_orbit = np.floor(ideal).astype(int)
    short = n - per_orbit.sum()
    per_orbit[np.argsort(-(ideal - per_orbit), kind="stable")[:short]] += 1
    pts = np.empty((n, 3))
    at = 0
    golden = 0.618033988749895
    for t, cnt in enumerate(per_orbit):
        if cnt == 0:
            continue
        az = 2.0 * math.pi * (np.arange(cnt) + (t * golden) % 1.0) / cnt
        s, z = math.sin(polar[t]), math.cos(polar[t])
        pts[at:at + cnt, 0] = s * np.cos(az)
        pts[at:at + cnt, 1] = s * np.sin(az)
        pts[at:at + cnt, 2] = z
        at += cnt
    pts /= np.linalg.norm(pts, axis=1, keepdims=True)
    return SampleSphere(pts, mode)


@dataclass
class ExposureStates:
    counts: np.ndarray    # uint8 0/1/2 per (atom, sample)
    critical: np.ndarray  # int32 coverer where count == 1, else -1


@dataclass(frozen=True)
class SasaResult:
    f_exp: np.ndarray
    a_exp: np.ndarray
    g_cav: float


def offset_radii(params, config: SolvationConfig) -> np.ndarray:
    return params.R + config.probe_radius


def check_cav_cutoff(params, config: SolvationConfig, d_cut_cav: float) -> None:
    """Setup check 2 (R_max + probe) <= d_cav (solvation.py:119-126)."""
    needed = 2.0 * (float(np.max(params.R)) + config.probe_radius)
    if needed > d_cut_cav:
        raise ConfigurationError(
            f"cavity cutoff {d_cut_cav} A below 2(R_max + probe) = {needed:.2f} A")


def force_quantum(params, r_off: np.ndarray, nq: int, delta_r: float):
    """Integer event magnitudes and the power-of-two quantum (solvation.py:184-191)."""
    delta = 4.0 * math.pi * params.gamma * r_off * r_off / (nq * delta_r)
    peak = float(np.max(np.abs(delta))) if len(delta) else 0.0
    if peak == 0.0:
        return np.zeros(len(delta), np.int64), 1.0
    quantum = 2.0 ** (math.floor(math.log2(peak)) - FIXED_POINT_BITS)
    return np.round(delta / quantum).astype(np.int64), quantum


# the reference's private name (solvation.py:184), kept for code written against it
_force_quantum = force_quantum


def sample_groups(points: np.ndarray, size: int = 32):
    """Order the sample directions into compact groups of <= `size` for the hot
    solvation kernel (one warp per group, lane = sample).

    Recursive bisection: each split sorts the set along one of 12 directions in
    the plane of its two principal axes, cuts at a multiple of `size`, and keeps
    the direction whose halves have the smaller angular radius.  Returns
    (groups: list of index arrays, cones: float32 [G, 8] = axis xyz, cos alpha,
    sin alpha, count, 0, 0), alpha bounding every member's angle to the axis.
    Coverage results do not depend on the sample order, so
    this is a pure scheduling choice."""
    pts = np.asarray(points, float)

    def radius(ix):
        a = pts[ix].mean(axis=0)
        a = a / max(float(np.linalg.norm(a)), 1e-12)
        return float(np.arccos(np.clip((pts[ix] @ a).min(), -1.0, 1.0)))

    groups = []

    def split(ix):
        if len(ix) <= size:
            groups.append(ix)
            return
        c = pts[ix] - pts[ix].mean(axis=0)
        v = np.linalg.svd(c, full_matrices=False)[2]
        half = ((len(ix) + size - 1) // size + 1) // 2 * size
        best = None
        for ang in np.linspace(0.0, np.pi, 12, endpoint=False):
            order = ix[np.argsort(c @ (np.cos(ang) * v[0] + np.sin(ang) * v[1]), kind="stable")]
            cost = max(radius(order[:half]), radius(order[half:]))
            if best is None or cost < best[0]:
                best = (cost, order)
        split(best[1][:half])
        split(best[1][half:])

    split(np.arange(len(pts)))
    cones = np.zeros((len(groups), 8), np.float32)
    for g, ix in enumerate(groups):
        a = pts[ix].mean(axis=0)
        norm = float(np.linalg.norm(a))
        if norm < 1e-6:                      # a group spread over the whole sphere
            a, ca = np.array([1.0, 0.0, 0.0]), -1.0
        else:
            a = a / norm
            ca = max(-1.0, float((pts[ix] @ a).min()) - 1e-6)
        cones[g, :3] = a
        cones[g, 3] = ca
        cones[g, 4] = math.sqrt(max(0.0, 1.0 - ca * ca))
        cones[g, 5] = len(ix)
    return groups, cones


def sasa_pass(positions, params, neighbors, sphere: SampleSphere,
              config: SolvationConfig = SolvationConfig()):
    from . import device
    return device.sasa_pass(positions, params, neighbors, sphere, config)


def solvation_forces(positions, params, neighbors, sphere: SampleSphere,
                     states: ExposureStates,
                     config: SolvationConfig = SolvationConfig()) -> np.ndarray:
    from . import device
    return device.solvation_forces(positions, params, neighbors, sphere, states, config)
