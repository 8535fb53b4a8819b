"""Spatial hash and cut-off neighbour tables: types and the drop-in API.

Types mirror /root/reference/pkg/src/kinefold/spatial.py:24-140.  The API
functions run on the GPU: ``build_grid`` (spatial.py:83-114) reduces the
bounding box on the device, derives the cell edge on the host with the
reference's own float expression (Python ``** (1/3)`` is not ``cbrt``, so the
edge must come from the same host arithmetic to be bit-identical), then bins
and sorts on the device; ``build_neighbor_table`` (spatial.py:163-230),
``filtered_pairs`` / ``filtered_lists`` (:233-259) likewise.  The KCM loop
itself never materialises these tables: it bins into its own hash grid inside
the pair kernel (csrc/kf_grid.cu), which yields the identical pair sets.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigurationError

SQRT3 = float(np.sqrt(3.0))


@dataclass(frozen=True)
class Cutoffs:
    elec: float = 9.0
    vdw: float = 5.0
    cav: float = 8.0

    def __post_init__(self):
        if min(self.elec, self.vdw, self.cav) <= 0:
            raise ConfigurationError("cutoff distances must be positive")

    def largest(self) -> float:
        return max(self.elec, self.vdw, self.cav)


@dataclass(frozen=True)
class GridConfig:
    alpha: float = 1.0
    min_cell: float = 1.0
    cutoffs: Cutoffs = field(default_factory=Cutoffs)

    def __post_init__(self):
        if self.alpha <= 0:
            raise ConfigurationError("alpha must be positive")


@dataclass
class HashGrid:
    cell_size: float
    r_min: np.ndarray
    r_max: np.ndarray
    dims: np.ndarray
    cell_index: np.ndarray
    _occupied: np.ndarray = field(repr=False)
    _starts: np.ndarray = field(repr=False)
    _atom_order: np.ndarray = field(repr=False)
    positions: np.ndarray = field(repr=False)

    @property
    def n_atoms(self) -> int:
        return len(self._atom_order)

    def linear_ids(self, cells: np.ndarray) -> np.ndarray:
        d = self.dims
        return (cells[..., 0] * d[1] + cells[..., 1]) * d[2] + cells[..., 2]

    @property
    def buckets(self) -> dict:
        out = {}
        d1, d2 = int(self.dims[1]), int(self.dims[2])
        for k, lin in enumerate(self._occupied):
            lin = int(lin)
            key = (lin // (d1 * d2), (lin // d2) % d1, lin % d2)
            out[key] = self._atom_order[self._starts[k]:self._starts[k + 1]]
        return out


@dataclass
class NeighborTable:
    """Per-atom superset neighbour rows, CSR (spatial.py:117-140)."""

    d_cut: float
    offsets: np.ndarray
    neighbors: np.ndarray

    @property
    def n_atoms(self) -> int:
        return len(self.offsets) - 1

    def list_of(self, i: int) -> np.ndarray:
        return self.neighbors[self.offsets[i]:self.offsets[i + 1]]

    def lists(self) -> list:
        return [self.list_of(i) for i in range(self.n_atoms)]

    def pairs(self):
        i = np.repeat(np.arange(self.n_atoms), np.diff(self.offsets))
        keep = self.neighbors > i
        return i[keep], self.neighbors[keep]


def reference_cell_edge(r_min, r_max, n: int, config: GridConfig):
    """Cell edge and dims with the reference's host float expression
    (spatial.py:92-96); inputs are the device-reduced exact min / max."""
    extent = r_max - r_min
    v_bb = float(np.prod(extent))
    cell = (v_bb / (config.alpha * n)) ** (1.0 / 3.0) if v_bb > 0 else 0.0
    cell = max(cell, config.min_cell)
    dims = np.maximum(np.ceil(extent / cell).astype(np.int64), 1)
    return float(cell), dims


def reference_stencil(cell: float, d_cut: float) -> np.ndarray:
    """Cell offsets whose centres lie within d_cut + sqrt(3) cell (spatial.py:143-151)."""
    r_c = d_cut + SQRT3 * cell
    reach = int(np.floor(r_c / cell))
    rng = np.arange(-reach, reach + 1)
    ox, oy, oz = np.meshgrid(rng, rng, rng, indexing="ij")
    offs = np.stack([ox.ravel(), oy.ravel(), oz.ravel()], axis=1)
    keep = (offs.astype(float) ** 2).sum(axis=1) * cell * cell <= r_c * r_c
    return offs[keep]


def build_grid(positions, config: GridConfig = GridConfig()) -> HashGrid:
    from . import device
    return device.build_grid(positions, config)


def build_neighbor_table(grid: HashGrid, d_cut: float) -> NeighborTable:
    from . import device
    return device.build_neighbor_table(grid, d_cut)


def filtered_pairs(table: NeighborTable, positions, d_cut: float):
    from . import device
    return device.filtered_pairs(table, positions, d_cut)


def filtered_lists(table: NeighborTable, positions, d_cut: float) -> list:
    from . import device
    return device.filtered_lists(table, positions, d_cut)


def brute_force_pairs(positions, d_cut: float):
    """All-pairs scan (the quadratic baseline, spatial.py:262-272): a full
    table of every other atom, filtered on the device."""
    positions = np.asarray(positions, float)
    n = len(positions)
    table = NeighborTable(float(d_cut), np.arange(n + 1, dtype=np.int64) * max(n - 1, 0),
                          _all_others(n))
    return filtered_pairs(table, positions, d_cut)


def _all_others(n: int) -> np.ndarray:
    if n < 2:
        return np.empty(0, np.int64)
    idx = np.arange(n, dtype=np.int64)
    full = np.broadcast_to(idx, (n, n))
    return full[~np.eye(n, dtype=bool)].reshape(-1)
