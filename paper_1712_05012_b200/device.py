"""Host side of the C ABI: device tables, batch buffers and every API call.

PyTorch is used only as the device allocator and stream provider; all
arithmetic on the hot path happens in libkfb200.so (include/kfb200.h).  Each
function here marshals the reference API's numpy arguments into device
tensors, fills the ABI structs, launches, and maps the device status block
back to the reference's exceptions and messages.

Caches: static chain / field tables are uploaded once per object (keyed by
identity plus a fingerprint of the arrays they were built from, so a mutated
chain is re-uploaded) and per-shape batch workspaces are reused.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time
import weakref
import zlib
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import (ConfigurationError, NativeLibraryError, StericClashError)
from .forcefield import MIN_DISTANCE, EnergyBreakdown
from .solvation import ExposureStates, SasaResult, check_cav_cutoff, force_quantum, sample_groups

_streams: dict = {}
_precision = {"pair": os.environ.get("KFB200_PAIR_PRECISION", "fp32")}


def set_pair_precision(mode: str) -> None:
    """Pair-kernel arithmetic: "fp32" (fp32 pair math, fp64 sums; the default)
    or "fp64" (reference formulas in fp64 for every pair: strict trajectory
    parity).  Membership decisions, solvation, FK, torques and the step are
    fp64 / exact in both modes."""
    if mode not in ("fp32", "fp64"):
        raise ConfigurationError(f"pair precision must be fp32 or fp64, got {mode!r}")
    _precision["pair"] = mode


def pair_precision() -> str:
    return _precision["pair"]


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise NativeLibraryError("no CUDA device: this package runs only on the GPU "
                                 "(there is no CPU path)")
    N.lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> torch.cuda.Stream:
    dev = _device()
    s = _streams.get(dev.index)
    if s is None:
        s = _streams[dev.index] = torch.cuda.Stream(device=dev)
    return s


def _sp():
    return C.c_void_p(stream().cuda_stream)


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _up(arr, dtype):
    """Host array -> device tensor on the package stream."""
    a = np.ascontiguousarray(arr, dtype=dtype)
    t = torch.from_numpy(a.copy() if not a.flags.writeable else a)
    return t.to(_device(), non_blocking=False)


def _call(name: str, *args) -> None:
    N.check(getattr(N.lib(), name)(*args), name)


def _fingerprint(*arrays) -> int:
    h = 0
    for a in arrays:
        a = np.ascontiguousarray(a)
        h = zlib.crc32(a.view(np.uint8).reshape(-1), h)
        h = zlib.crc32(str(a.shape).encode(), h)
    return h


class _IdCache:
    """id(obj) -> (weakref, fingerprint, value); stale entries are rebuilt."""

    def __init__(self):
        self._d = {}

    def get(self, obj, fp, build):
        key = id(obj)
        hit = self._d.get(key)
        if hit is not None:
            ref, hfp, val = hit
            if ref() is obj and hfp == fp:
                return val
        val = build()
        try:
            ref = weakref.ref(obj)
        except TypeError:
            ref = (lambda o: (lambda: o))(obj)
        self._d[key] = (ref, fp, val)
        if len(self._d) > 64:
            for k in list(self._d)[:-32]:
                del self._d[k]
        return val


_chain_cache = _IdCache()
_field_cache = _IdCache()
_tree_cache = _IdCache()


# --------------------------------------------------------------------------
# static chain tables
# --------------------------------------------------------------------------

class DeviceChain:
    """Link tree, FK / torque schedules and atom tables of one chain (kf_chain_t)."""

    def __init__(self, chain):
        links = list(chain.links)
        L = len(links)
        n = int(len(chain.atom_link))
        D = L - 1
        R = int(chain.n_residues)
        if L < 1 or links[0].kind != "ground":
            raise ConfigurationError("link 0 must be the ground link")
        parent = np.array([l.parent for l in links], np.int64)
        dof = np.array([l.dof for l in links], np.int64)
        if np.any(parent[1:] >= np.arange(1, L)) or np.any(parent[1:] < 0):
            raise ConfigurationError("links must be topologically ordered (parent < index)")
        if sorted(dof[1:].tolist()) != list(range(D)):
            raise ConfigurationError("non-ground links must carry dofs 0..n_dof-1")
        axis0 = np.zeros((L, 3))
        body0 = np.zeros((L, 3))
        point0 = np.zeros((L, 3))
        for k, l in enumerate(links):
            if l.axis0 is not None:
                axis0[k] = l.axis0
            body0[k] = l.body0
            point0[k] = l.point0
        kinds = [l.kind for l in links]
        bb = sorted((k for k in range(L) if kinds[k] in ("phi", "psi")), key=lambda k: dof[k])
        prev = 0
        for k in bb:
            if parent[k] != prev:
                raise ConfigurationError("backbone (phi/psi) links must form a path from ground")
            prev = k
        if sorted(int(dof[k]) for k in bb) != list(range(len(bb))):
            raise ConfigurationError("backbone links must carry dofs 0..2m-1 (side links after)")
        bb_set = set(bb)
        depth = np.zeros(L, np.int64)
        side = []
        for k in range(1, L):
            if k in bb_set:
                continue
            depth[k] = depth[parent[k]] + 1 if parent[k] not in bb_set and parent[k] != 0 else 1
            side.append(k)
        side.sort(key=lambda k: (depth[k], k))
        max_depth = int(depth.max()) if side else 0
        side_depth_off = np.searchsorted(depth[side] if side else np.zeros(0, np.int64),
                                         np.arange(1, max_depth + 2))
        chi_by_res = [[] for _ in range(R)]
        for k, l in enumerate(links):
            if l.kind == "chi":
                if not 0 <= l.residue < R:
                    raise ConfigurationError(f"chi link {k} has residue {l.residue} out of range")
                chi_by_res[l.residue].append(k)
        for lst in chi_by_res:
            lst.sort(key=lambda k: links[k].chi_index)
        chi_off = np.concatenate([[0], np.cumsum([len(x) for x in chi_by_res])]).astype(np.int64)
        chi_links = np.array([k for x in chi_by_res for k in x], np.int64)
        bb_side_res = np.array([links[k].residue if kinds[k] == "phi" else -1 for k in bb], np.int64)
        atom_link = np.asarray(chain.atom_link, np.int64)
        zp = np.asarray(chain.zp_pos, float)
        zrel = zp - point0[atom_link]
        order = np.argsort(atom_link, kind="stable")
        link_off = np.concatenate([[0], np.cumsum(np.bincount(atom_link, minlength=L))])

        self.n_atoms, self.n_links, self.n_dof, self.n_res = n, L, D, R
        self.n_bb = len(bb)
        self.bb_links = np.array(bb, np.int64)
        i32 = np.int32
        t = self.tensors = dict(
            link_parent=_up(np.maximum(parent, 0), i32), link_dof=_up(dof, i32),
            link_axis0=_up(axis0, np.float64), link_body0=_up(body0, np.float64),
            bb_order=_up(bb, i32), side_order=_up(side, i32),
            side_depth_off=_up(side_depth_off, i32), atom_link=_up(atom_link, i32),
            atom_zrel=_up(zrel, np.float64), link_atom_off=_up(link_off, i32),
            link_atoms=_up(order, i32), chi_res_off=_up(chi_off, i32),
            chi_links=_up(chi_links, i32), bb_by_dof=_up(bb, i32),
            bb_side_res=_up(bb_side_res, i32))
        s = self.struct = N.KfChain()
        s.n_atoms, s.n_links, s.n_dof, s.n_res = n, L, D, R
        s.n_bb, s.n_side, s.side_depth = len(bb), len(side), max_depth
        for name, ten in t.items():
            setattr(s, name, ten.data_ptr() if ten.numel() else None)
        self._fk_batch = None

    def fk_batch(self):
        if self._fk_batch is None:
            self._fk_batch = Batch(self, None, 1)
        return self._fk_batch


def device_chain(chain) -> DeviceChain:
    fp = _fingerprint(np.asarray(chain.zp_pos, float), np.asarray(chain.atom_link),
                      np.array([len(chain.links)]))
    return _chain_cache.get(chain, fp, lambda: DeviceChain(chain))


# --------------------------------------------------------------------------
# static field tables
# --------------------------------------------------------------------------

def _sqrt_threshold(cut: float) -> float:
    """Largest d2 with sqrt(d2) <= cut, so `d2 <= thr` == `sqrt(d2) <= cut`
    exactly (the reference compares d = sqrt(d2) with the per-term cutoff,
    kcm.py:115, :120)."""
    cut = float(cut)
    x = cut * cut
    while np.sqrt(np.nextafter(x, np.inf)) <= cut:
        x = float(np.nextafter(x, np.inf))
    while np.sqrt(x) > cut:
        x = float(np.nextafter(x, -np.inf))
    return float(x)


def _stencil(cell: float, reach_dist: float) -> np.ndarray:
    """The 27 offsets of a one-cell reach: own cell, the 13 lexicographically
    positive offsets, then their negatives (a half-shell order, kept so a
    Newton's-third-law pair kernel can take the first 14)."""
    if cell < reach_dist:
        raise ConfigurationError("hot-path cells must be at least one interaction reach wide")
    rng = np.arange(-1, 2)
    ox, oy, oz = np.meshgrid(rng, rng, rng, indexing="ij")
    offs = np.stack([ox.ravel(), oy.ravel(), oz.ravel()], axis=1)
    fwd = [tuple(o) for o in offs if tuple(o) > (0, 0, 0)]
    bwd = [tuple(-np.array(o)) for o in fwd]
    return np.array([(0, 0, 0)] + fwd + bwd, dtype=np.int64)


def tree_classes(tree, i, j) -> np.ndarray:
    """Reference interaction classes of pairs (topology.py:153-178), host numpy;
    used only to build the static per-atom class window below."""
    p, gp, gg = (np.asarray(a, np.int64) for a in (tree.parent, tree.grandparent, tree.greatgrand))
    res = np.asarray(tree.residue_of, np.int64)
    chain = np.asarray(tree.chain_mask, bool)
    eq = lambda a, b: (a == b) & (a >= 0)  # noqa: E731
    near = chain[i] & chain[j] & (np.abs(res[i] - res[j]) <= 1)
    c = np.full(len(i), 4, np.int64)
    c[near & (eq(gg[i], j) | eq(gg[j], i) | eq(gp[i], p[j]) | eq(gp[j], p[i]))] = 3
    c[near & (eq(gp[i], j) | eq(gp[j], i) | eq(p[i], p[j]))] = 2
    c[near & (eq(p[i], j) | eq(p[j], i))] = 1
    return c


def class_window(tree):
    """Static topology table for the pair kernel: per atom, 2-bit codes
    (4 - class) for partners j = i-32 .. i+31 packed in 4 int32 words, and a
    flag for atoms with a class < 4 partner outside the window (those fall
    back to the tree predicate on the device)."""
    n = len(tree.parent)
    off = np.arange(64) - 32
    ii = np.repeat(np.arange(n), 64)
    jj = ii + np.tile(off, n)
    ok = (jj >= 0) & (jj < n) & (jj != ii)
    codes = np.zeros(n * 64, np.uint64)
    c = tree_classes(tree, ii[ok], jj[ok])
    codes[ok] = (4 - c).astype(np.uint64)
    codes = codes.reshape(n, 4, 16)
    words = (codes << (2 * np.arange(16, dtype=np.uint64))).sum(axis=2).astype(np.uint32)
    # partners beyond the window: same or adjacent residue, any index distance
    slow = np.zeros(n, bool)
    res = np.asarray(tree.residue_of, np.int64)
    chain = np.asarray(tree.chain_mask, bool)
    order = np.argsort(res, kind="stable")
    bounds = np.searchsorted(res[order], np.unique(res))
    groups = np.split(order, bounds[1:])
    by_res = {int(res[g[0]]): g for g in groups if len(g)}
    for r, g in by_res.items():
        nb = np.concatenate([by_res.get(r + d, np.zeros(0, np.int64)) for d in (0, 1)])
        a = np.repeat(g, len(nb))
        b = np.tile(nb, len(g))
        far = (np.abs(a - b) >= 32) & chain[a] & chain[b]
        if far.any():
            cc = tree_classes(tree, a[far], b[far])
            hit = cc < 4
            slow[a[far][hit]] = True
            slow[b[far][hit]] = True
    return words.view(np.int32), slow


def class_codes(tree) -> np.ndarray:
    """Static pair classes for the cluster-pair kernel (kf_cluster.cu): for quad Q
    (atoms 4Q..4Q+3) and the octets O = Q//2 + k, k = 0..4, a uint64 of 2-bit
    (4 - class) codes, pair (i = 4Q + l % 4, j = 8O + l // 4) at bits 2l.  These
    octets hold every partner within the 64-atom window of the quad; partners
    beyond it are class 4 except for class_window's slow atoms."""
    n = len(tree.parent)
    nq = (n + 3) // 4
    lane = np.arange(32)
    Q = np.repeat(np.arange(nq), 5)
    k = np.tile(np.arange(5), nq)
    i = (4 * Q)[:, None] + (lane % 4)[None, :]
    j = (8 * (Q // 2 + k))[:, None] + (lane // 4)[None, :]
    ok = (i < n) & (j < n) & (j != i)
    c = np.full(i.shape, 4, np.int64)
    c[ok] = tree_classes(tree, i[ok], j[ok])
    code = ((4 - c).astype(np.uint64) << (2 * lane).astype(np.uint64)[None, :]).sum(axis=1, dtype=np.uint64)
    return code.reshape(nq, 5)


def unit_codes(codes, slow) -> np.ndarray:
    """class_codes regrouped per (unit U = quads 2U, 2U+1; lane l) as the cluster
    kernel's lanes use them (kfb200.h unit_codes): one coalesced 32-bit load per
    lane and unit instead of 10 code words and the slow-atom flags."""
    nq = codes.shape[0]
    no = (nq + 1) // 2
    c = np.zeros((2 * no, 5), np.uint64)
    c[:nq] = codes
    lane = np.arange(32, dtype=np.uint64)
    bits = (c[:, :, None] >> (2 * lane)[None, None, :]) & np.uint64(3)      # [2 no][5][32]
    k2 = (2 * np.arange(5, dtype=np.uint64))[:, None]
    qa = (bits[0::2] << k2).sum(axis=1, dtype=np.uint64)                       # [no][32]
    qb = (bits[1::2] << (k2 + np.uint64(10))).sum(axis=1, dtype=np.uint64)
    nz = (c != 0).astype(np.uint64)
    win = ((nz[0::2] << np.arange(5, dtype=np.uint64)).sum(axis=1, dtype=np.uint64) << np.uint64(20)) | \
          ((nz[1::2] << np.arange(5, dtype=np.uint64)).sum(axis=1, dtype=np.uint64) << np.uint64(25))
    n = len(slow)
    s = np.zeros(8 * no, bool)
    s[:n] = slow
    su = s.reshape(no, 8).any(axis=1).astype(np.uint64) << np.uint64(30)
    return (qa | qb | (win | su)[:, None]).astype(np.uint32)


class ParamTables:
    """Per-atom parameters + pair-weight provider + dielectric on the device."""

    def __init__(self, params, weights, dielectric, n: int):
        q = np.asarray(params.q, float)
        if len(q) != n:
            raise ConfigurationError(f"parameters cover {len(q)} atoms, positions have {n}")
        R = np.asarray(params.R, float)
        eps = np.asarray(params.eps, float)
        gamma = np.asarray(params.gamma, float)
        f32 = np.float32
        t = self.tensors = dict(q32=_up(q, f32), R32=_up(R, f32), seps32=_up(np.sqrt(eps), f32),
                                q=_up(q, np.float64), R=_up(R, np.float64), eps=_up(eps, np.float64))
        s = self.struct = N.KfField()
        s.n_atoms = n
        par = np.zeros((n, 4), f32)
        par[:, 0], par[:, 1], par[:, 2] = q, R, np.sqrt(eps)
        aux = np.zeros((n, 4), np.int32)
        aux[:, 0] = np.arange(n)
        if hasattr(weights, "tree") and hasattr(weights, "table"):
            aux[:, 1] = np.asarray(weights.tree.residue_of)
            aux[:, 2] = np.asarray(weights.tree.chain_mask).astype(np.int32)
            tree = weights.tree
            cmap, slow = class_window(tree)
            t.update(tparent=_up(tree.parent, np.int32), tgp=_up(tree.grandparent, np.int32),
                     tggp=_up(tree.greatgrand, np.int32), tres=_up(tree.residue_of, np.int32),
                     tchain=_up(tree.chain_mask, np.uint8), class_map=_up(cmap, np.int32),
                     class_slow=_up(slow, np.uint8),
                     class_codes=_up(class_codes(tree).view(np.int64), np.int64))
            t.update(unit_codes=_up(unit_codes(class_codes(tree), slow).view(np.int32), np.int32))
            aux[:, 3] = slow.astype(np.int32)
            s.uniform_weights = 0
            for k, v in enumerate(np.asarray(weights.table.elec_by_class())[1:5]):
                s.w_elec[k] = float(v)
            for k, v in enumerate(np.asarray(weights.table.vdw_by_class())[1:5]):
                s.w_vdw[k] = float(v)
        elif hasattr(weights, "value") and type(weights).__name__ == "UniformWeights":
            s.uniform_weights = 1
            s.uniform_value = float(weights.value)
        else:
            raise ConfigurationError(
                f"unsupported pair-weight provider {type(weights).__name__}: "
                "use TreeWeights or UniformWeights")
        t.update(atom_par=_up(par, f32), atom_aux=_up(aux, np.int32))
        if dielectric is not None:
            s.dielectric_const = 1 if dielectric.mode == "constant" else 0
            s.kappa = float(dielectric.kappa)
        for name, ten in t.items():
            setattr(s, name, ten.data_ptr())


class DeviceField(ParamTables):
    """Everything kf_field_t carries for one Field (cut-offs, hash grid, solvation)."""

    def __init__(self, fld, n: int):
        cfg = fld.config
        super().__init__(fld.params, fld.weights, cfg.dielectric, n)
        s, t = self.struct, self.tensors
        cut = cfg.cutoffs
        cut_pair = max(cut.elec, cut.vdw)
        s.cut_pair2 = cut_pair * cut_pair
        s.thr_elec2 = _sqrt_threshold(cut.elec)
        s.thr_vdw2 = _sqrt_threshold(cut.vdw)
        reach = float(cut_pair)
        self.solvation = bool(cfg.solvation)
        s.solvation = int(self.solvation)
        if self.solvation:
            scfg = cfg.solvation_cfg
            sphere = fld.sphere()
            r_off = np.asarray(fld.params.R, float) + scfg.probe_radius
            r_off2 = r_off * r_off
            w_int, quantum = force_quantum(fld.params, r_off, sphere.n, scfg.delta_r)
            gamma = np.asarray(fld.params.gamma, float)
            s.reach_pad = scfg.delta_r + 1e-3
            s.r_off_max = float(np.max(r_off)) if len(r_off) else 0.0
            reach = max(reach, 2.0 * float(np.max(r_off)) + s.reach_pad)
            t.update(samples=_up(sphere.points, np.float64), r_off=_up(r_off, np.float64),
                     r_off2=_up(r_off2, np.float64), gamma=_up(gamma, np.float64),
                     w_int=_up(w_int, np.int64),
                     solv_nz=_up(np.flatnonzero(gamma != 0.0), np.int32),
                     solv_all=_up(np.arange(n), np.int32))
            s.n_samples = sphere.n
            groups, cones = sample_groups(sphere.points)
            grp = np.zeros((len(groups), 32, 3))
            for g, ix in enumerate(groups):
                grp[g, :len(ix)] = np.asarray(sphere.points, float)[ix]
            t.update(samples_grp=_up(grp, np.float64), grp_cone=_up(cones, np.float32))
            s.samples_grp, s.grp_cone = t["samples_grp"].data_ptr(), t["grp_cone"].data_ptr()
            s.n_groups = len(groups)
            s.quantum, s.delta_r, s.four_pi = float(quantum), float(scfg.delta_r), 4.0 * math.pi
            for name in ("samples", "r_off", "r_off2", "gamma", "w_int"):
                setattr(s, name, t[name].data_ptr())
            self.n_solv_nz = int(np.count_nonzero(gamma != 0.0))
        reach *= 1.0 + 1e-9
        s.cell = reach              # one cell per reach: the 27-cell stencil
        # use_hash=False (kcm.py:94-102): one all-atom cell, every pair a candidate
        s.flat = 0 if cfg.use_hash else 1
        sten = _stencil(s.cell, reach) if cfg.use_hash else np.zeros((1, 3), np.int64)
        t["stencil"] = _up(sten, np.int32)
        s.stencil = t["stencil"].data_ptr()
        s.n_stencil = len(sten)
        assert s.n_stencil <= 32, "one-cell reach stencil expected (27 cells)"
        # H > n buckets: room for the worst case (one cell per atom) with one empty slot
        # to end every probe, and for the item -> cell map (items <= n)
        s.hash_bits = max(6, int(math.ceil(math.log2(n + 1))))
        s.precision = 1 if _precision["pair"] == "fp64" else 0
        self.n = n
        self._batches = {}

    def struct_for(self, all_atoms: bool) -> N.KfField:
        """kf_field_t with the solvation atom list: every atom (API results need
        f_exp of all atoms) or only gamma != 0 atoms (the fold loop)."""
        s = N.KfField()
        C.pointer(s)[0] = self.struct
        if self.solvation:
            key = "solv_all" if all_atoms else "solv_nz"
            s.solv_atoms = self.tensors[key].data_ptr() if self.tensors[key].numel() else None
            s.n_solv = self.n if all_atoms else self.n_solv_nz
        return s

    def batch(self, chain_dev, B: int, **kw):
        key = (id(chain_dev), B, tuple(sorted(kw.items())))
        b = self._batches.get(key)
        if b is None:
            if len(self._batches) > 8:
                self._batches.clear()
            b = self._batches[key] = Batch(chain_dev, self, B, **kw)
        return b


def device_field(fld, n: int) -> DeviceField:
    p = fld.params
    fp = _fingerprint(np.asarray(p.q, float), np.asarray(p.R, float), np.asarray(p.eps, float),
                      np.asarray(p.gamma, float), np.array([n])) ^ hash(repr(fld.config)) ^ id(fld.weights) \
        ^ hash(_precision["pair"])
    return _field_cache.get(fld, fp, lambda: DeviceField(fld, n))


# --------------------------------------------------------------------------
# batch workspace
# --------------------------------------------------------------------------

class Batch:
    """Per-iteration buffers for B trajectories (kf_batch_t)."""

    def __init__(self, dc: DeviceChain | None, df: DeviceField | None, B: int, *,
                 max_records: int = 0, record_theta: bool = False, store_sasa: bool = False,
                 nb_cap: int | None = None):
        dev = _device()
        if nb_cap is None:
            nb_cap = int(os.environ.get("KFB200_SOLV_NB_CAP", "512"))
        n = dc.n_atoms if dc is not None else df.n
        L = dc.n_links if dc is not None else 1
        D = dc.n_dof if dc is not None else 0
        R = dc.n_res if dc is not None else 0
        nbb = dc.n_bb if dc is not None else 0
        H = 1 << (df.struct.hash_bits if df is not None else 6)
        f64, i32 = torch.float64, torch.int32
        z = lambda *shape, dtype=f64: torch.zeros(*shape, dtype=dtype, device=dev)  # noqa: E731
        with torch.cuda.stream(stream()):
            t = self.t = dict(
                theta=z(B, max(D, 1)), frozen=z(B, max(D, 1), dtype=torch.uint8),
                link_T=z(B, L, 16), fk_scratch=z(B, max(1, -(-nbb // 256)), 12),   # >= ceil(n_bb / segment) rows
                pos=z(B, n, 3), forces=z(B, n, 3),
                cell_key=z(B, H, dtype=torch.int64), cell_cnt=z(B, H, dtype=i32),
                cell_start=z(B, H, dtype=i32), occ=z(B, H, dtype=i32), occ_count=z(B, dtype=i32),
                occ_offset=z(B + 1, dtype=i32), chunk_pre=z(B, H, dtype=i32), item_cell=z(B, H, dtype=i32),
                chunk_count=z(B, dtype=i32), chunk_offset=z(B + 1, dtype=i32), atom_slot=z(B, n, dtype=i32), atom_rank=z(B, n, dtype=i32),
                sorted_atom=z(B, n, dtype=i32), s_hi=z(B, n, 4, dtype=torch.float32),
                s_lo=z(B, n, 4, dtype=torch.float32), s_pos=z(B, n, 4),
                s_par=z(B, n, 4, dtype=torch.float32), s_aux=z(B, n, 4, dtype=i32),
                s_tree=z(B, n, 4, dtype=i32), cell_box=z(B, H, 8, dtype=torch.float32),
                work=z(4, dtype=i32),
                e_atom=z(B, n, 2), pair_count=z(B, n, dtype=torch.int64),
                solv_acc=z(B, n, 3, dtype=torch.int64), solv_ovf=z(1 + 2 * B * n, dtype=i32),
                pair_fj=z(B, n, 9, dtype=torch.int64), cav_atom=z(B, n),
                f_exp=z(B, n) if store_sasa else None, a_exp=z(B, n) if store_sasa else None,
                wrench=z(B, L, 6), side_tot=z(B, max(R, 1), 6), bb_suffix=z(B, max(nbb, 1), 6),
                tau=z(B, max(D, 1)), energy=z(B, 3),
                status=z(B, C.sizeof(N.KfStatus), dtype=torch.uint8),
                rec_energy=z(B, max(max_records, 1), 4),
                rec_theta=z(B, max_records, max(D, 1)) if record_theta and max_records else None)
        s = self.struct = N.KfBatch()
        s.B, s.n_buckets, s.nb_cap = B, H, nb_cap
        s.record_theta = int(bool(record_theta and max_records))
        s.max_records = max_records
        for name, ten in t.items():
            setattr(s, name, ten.data_ptr() if ten is not None else None)
        self.B, self.n, self.D = B, n, D

    def reset_status(self):
        self.t["status"].zero_()
        # a trajectory stopped by a device error leaves its half-list fixed-point
        # j forces uncleared (the wrench pass that folds them in does not run)
        self.t["pair_fj"].zero_()

    def status(self):
        raw = self.t["status"].cpu().numpy().tobytes()
        return (N.KfStatus * self.B).from_buffer_copy(raw)

    def status_array(self) -> np.ndarray:
        """The status block as a numpy structured array (one D2H copy)."""
        return np.frombuffer(self.t["status"].cpu().numpy().tobytes(), np.dtype(N.KfStatus))

    def status_snapshots(self):
        """Two pinned host copies of the status block with their events (the
        fold loop's pipelined stop test)."""
        if getattr(self, "_snaps", None) is None:
            self._snaps = [(torch.empty_like(self.t["status"], device="cpu").pin_memory(),
                            torch.cuda.Event()) for _ in range(2)]
        return self._snaps


# --------------------------------------------------------------------------
# errors from the device status block
# --------------------------------------------------------------------------

def _raise_status(st, df: DeviceField | None, batch: Batch, prefix: str = "", b: int = 0):
    if st.error == N.ERR_CLASH:
        fs = df.struct_for(False)
        _call("kf_clash_report", N.ref(fs), N.ref(batch.struct), _sp())
        st = batch.status()[b]
        i, j = int(st.clash_key >> 32), int(st.clash_key & 0xFFFFFFFF)
        d = float(np.frombuffer(np.uint64(st.dmin_bits).tobytes(), np.float64)[0])
        raise StericClashError(f"{prefix}atoms {i} and {j} closer than {MIN_DISTANCE} A (d={d:.3e})")
    if st.error == N.ERR_NONFINITE:
        raise ConfigurationError(f"{prefix}non-finite coordinates cannot be hashed")
    if st.error == N.ERR_EXTENT:
        raise ConfigurationError(f"{prefix}use_hash=False: an atom lies more than 2048 A from the structure's "
                                 "centroid cell (fp32 offset range of the all-pairs layout)")
    if st.error == N.ERR_CAPACITY:
        if st.overflow < 0:   # the cluster-pair kernel's exact-path queue (2 n pairs)
            raise NativeLibraryError(f"{prefix}{-st.overflow} pairs need the exact fp64 path, more than the "
                                     f"cluster-pair kernel's queue of {2 * batch.n}")
        raise NativeLibraryError(f"{prefix}solvation neighbour capacity exceeded "
                                 f"({st.overflow} > {batch.struct.nb_cap})")


def _prep_clash_key(batch: Batch):
    # dmin_bits and clash_key start at all-ones so atomicMin finds the
    # smallest distance and then the smallest (i, j) at that distance
    st = batch.t["status"].view(torch.uint8).reshape(batch.B, -1)
    for fld in (N.KfStatus.dmin_bits, N.KfStatus.clash_key):
        st[:, fld.offset:fld.offset + 8] = 0xFF


# --------------------------------------------------------------------------
# forward kinematics
# --------------------------------------------------------------------------

def kinematic_state(chain, theta, positions_only: bool = False):
    dc = device_chain(chain)
    b = dc.fk_batch()
    with torch.cuda.stream(stream()):
        b.t["theta"][0, :dc.n_dof].copy_(torch.from_numpy(np.asarray(theta, float)))
        _call("kf_fk", N.ref(dc.struct), N.ref(b.struct), _sp())
        pos = b.t["pos"][0].cpu().numpy()
        if positions_only:
            return pos
        T = b.t["link_T"][0].cpu().numpy()
    M = T[:, :9].reshape(-1, 3, 3)
    return M, T[:, 9:12].copy(), T[:, 12:15].copy(), pos


# --------------------------------------------------------------------------
# Field.evaluate
# --------------------------------------------------------------------------

def _positions(positions) -> np.ndarray:
    pos = np.asarray(positions, float)
    if pos.ndim != 2 or pos.shape[1] != 3 or len(pos) < 1:
        raise ConfigurationError("positions must be a non-empty (n, 3) array")
    return pos


def evaluate(fld, positions, *, energy_only: bool = False):
    from .kcm import FieldResult
    pos = _positions(positions)
    n = len(pos)
    df = device_field(fld, n)
    if df.solvation:
        check_cav_cutoff(fld.params, fld.config.solvation_cfg, fld.config.cutoffs.cav)
    b = df.batch(None, 1, store_sasa=df.solvation)
    b.struct.api_eval = 1
    fs = df.struct_for(True)
    s = stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    with torch.cuda.stream(s):
        b.reset_status()
        _prep_clash_key(b)
        b.t["pos"][0].copy_(torch.from_numpy(pos))
        ev[0].record(s)
        _call("kf_bin", N.ref(fs), N.ref(b.struct), _sp())
        ev[1].record(s)
        _call("kf_pairs", N.ref(fs), N.ref(b.struct), _sp())
        ev[2].record(s)
        if df.solvation:
            _call("kf_solvation", N.ref(fs), N.ref(b.struct), _sp())
        _call("kf_energy_reduce", N.ref(fs), N.ref(b.struct), n, _sp())
        ev[3].record(s)
        st = b.status()[0]
        if st.error:
            _raise_status(st, df, b)
        e = b.t["energy"][0].cpu().numpy()
        forces = np.zeros((n, 3)) if energy_only else b.t["forces"][0].cpu().numpy()
        sasa = None
        if df.solvation:
            sasa = SasaResult(b.t["f_exp"][0].cpu().numpy(), b.t["a_exp"][0].cpu().numpy(), float(e[2]))
    s.synchronize()
    ms = lambda a, c: ev[a].elapsed_time(ev[c]) * 1e-3  # noqa: E731
    timings = {"hash": ms(0, 1), "force": ms(1, 2), "solvation": ms(2, 3) if df.solvation else 0.0}
    return FieldResult(forces=forces, energy=EnergyBreakdown(float(e[0]), float(e[1]), float(e[2])),
                       timings=timings, sasa=sasa)


# --------------------------------------------------------------------------
# the fold loop
# --------------------------------------------------------------------------

def _step_struct(step) -> N.KfStep:
    s = N.KfStep()
    s.kappa, s.torque_tol, s.torque_tol_rel = float(step.kappa), float(step.torque_tol), float(step.torque_tol_rel)
    s.energy_tol, s.max_iters, s.energy_window = float(step.energy_tol), int(step.max_iters), int(step.energy_window)
    return s


_STATUS_DTYPE = np.dtype(N.KfStatus)


def _run_loop(dc, df, b, step, chunk: int, on_first=None):
    """Replay graph chunks until every trajectory reports done.  The stop test
    is pipelined: chunk k+1 is enqueued before the host reads chunk k's status
    (an async copy into pinned memory), so the GPU never idles on the poll; a
    chunk enqueued after the last trajectory stopped is a no-op on device."""
    lib = N.lib()
    cs, fs, bs, ss = N.ref(dc.struct), N.ref(df.struct_for(False)), N.ref(b.struct), N.ref(_step_struct(step))
    s = stream()
    done_iters = 0
    if on_first is not None and step.max_iters > 0:
        on_first(cs, fs, bs, ss)
        done_iters = 1
        if all(x.done for x in b.status()):
            done_iters = step.max_iters
    snaps = b.status_snapshots()
    pending, turn = None, 0
    while done_iters < step.max_iters:
        k = min(chunk, step.max_iters - done_iters)
        N.check(lib.kf_fold_iterations(cs, fs, bs, ss, k, _sp()), "kf_fold_iterations")
        done_iters += k
        if done_iters >= step.max_iters:
            break
        host, ev = snaps[turn]
        host.copy_(b.t["status"], non_blocking=True)
        ev.record(s)
        if pending is not None:
            p_host, p_ev = pending
            p_ev.synchronize()
            if np.frombuffer(p_host.numpy().tobytes(), _STATUS_DTYPE)["done"].all():
                break
        pending, turn = snaps[turn], 1 - turn
    s.synchronize()


def fold(chain, conf, fld, step):
    from .chain import Conformation
    from .kcm import IterationRecord, Trajectory
    chain_D = len(chain.links) - 1
    if np.asarray(conf.theta).shape[0] != chain_D:
        raise ConfigurationError(
            f"conformation has {np.asarray(conf.theta).shape[0]} dofs, chain needs {chain_D}")
    dc = device_chain(chain)
    n = dc.n_atoms
    df = device_field(fld, n)
    if df.solvation and step.max_iters > 0:
        try:
            check_cav_cutoff(fld.params, fld.config.solvation_cfg, fld.config.cutoffs.cav)
        except ConfigurationError as exc:
            raise ConfigurationError(f"aborted at iteration 0: {exc}") from exc
    K = int(step.max_iters)
    # one cached workspace per (chain, K): repeated folds reuse its buffers and
    # hence the CUDA graphs captured on them
    b = df.batch(dc, 1, max_records=K, record_theta=True)
    s = stream()
    phase = {}

    def first_iteration(cs, fs, bs, ss):
        # iteration 0 eagerly, with CUDA events between phases, to apportion
        # per-iteration wall time to the reference's phase names
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        lib = N.lib()
        ev[0].record(s)
        N.check(lib.kf_fk(cs, bs, _sp()), "kf_fk")
        ev[1].record(s)
        N.check(lib.kf_bin(fs, bs, _sp()), "kf_bin")
        ev[2].record(s)
        N.check(lib.kf_pairs(fs, bs, _sp()), "kf_pairs")
        ev[3].record(s)
        if df.solvation:
            N.check(lib.kf_solvation(fs, bs, _sp()), "kf_solvation")
        ev[4].record(s)
        N.check(lib.kf_torques_step(cs, fs, bs, ss, _sp()), "kf_torques_step")
        ev[5].record(s)
        s.synchronize()
        names = ["fk", "hash", "force", "solvation", "torque"]
        for k, nm in enumerate(names):
            phase[nm] = ev[k].elapsed_time(ev[k + 1]) * 1e-3

    with torch.cuda.stream(s):
        b.reset_status()
        _prep_clash_key(b)
        b.t["theta"][0].copy_(torch.from_numpy(np.asarray(conf.theta, float)))
        b.t["frozen"][0].copy_(torch.from_numpy(np.asarray(conf.frozen, np.uint8)))
        t0 = time.perf_counter()
        _run_loop(dc, df, b, step, chunk=16, on_first=first_iteration)
        wall = time.perf_counter() - t0
        st = b.status()[0]
        if st.error:
            _raise_status(st, df, b, prefix=f"aborted at iteration {st.err_iter}: ")
        iters = int(st.iter)
        rec = b.t["rec_energy"][0, :iters].cpu().numpy()
        thetas = b.t["rec_theta"][0, :iters].cpu().numpy() if iters else np.zeros((0, chain_D))
        final_theta = b.t["theta"][0, :chain_D].cpu().numpy()
    per_iter = wall / max(iters, 1)
    tot = sum(phase.values()) or 1.0
    timings = {k: per_iter * v / tot for k, v in phase.items()}
    if not df.solvation:
        timings["solvation"] = 0.0
    records, snapshots = [], []
    frozen = np.asarray(conf.frozen, bool)
    for k in range(iters):
        e = rec[k]
        records.append(IterationRecord(k, EnergyBreakdown(float(e[0]), float(e[1]), float(e[2])),
                                       float(e[3]), dict(timings), thetas[k].copy()))
        if step.snapshot_every and k % step.snapshot_every == 0:
            snapshots.append((k, Conformation(thetas[k].copy(), frozen, conf.residue_count)))
    reason = N.REASONS.get(int(st.reason), "max_iters")
    final = Conformation(final_theta, frozen, conf.residue_count)
    return Trajectory(records, snapshots, final, reason != "max_iters", reason)


@dataclass
class EnsembleResult:
    """Batched fold output (one chain, B trajectories)."""

    theta: np.ndarray        # [B, D] final dihedrals
    energies: np.ndarray     # [B, K, 4] g_elec, g_vdw, g_cav, tau_max per iteration
    iterations: np.ndarray   # [B]
    reasons: list
    thetas: np.ndarray | None = None   # [B, K, D] when recorded
    n_pairs: np.ndarray | None = None  # [B] pairs within the elec cutoff, last iteration

    @property
    def converged(self) -> np.ndarray:
        return np.array([r != "max_iters" for r in self.reasons])


class EnsembleRunner:
    """Reusable device state for repeated ensemble runs (bench and sharded runs)."""

    def __init__(self, chain, fld, B: int, step, *, record_theta: bool = False, chunk: int = 8):
        self.dc = device_chain(chain)
        self.df = device_field(fld, self.dc.n_atoms)
        self.B, self.step, self.chunk = B, step, chunk
        self.batch = Batch(self.dc, self.df, B, max_records=int(step.max_iters),
                           record_theta=record_theta)
        self.fld = fld

    def _pinned(self):
        if getattr(self, "_pin", None) is None:
            D = self.dc.n_dof
            self._pin = (torch.empty((self.B, D), dtype=torch.float64).pin_memory(),
                         torch.empty((self.B, D), dtype=torch.uint8).pin_memory())
        return self._pin

    def load(self, thetas, frozen):
        """Host conformations in: staged in pinned memory, copied asynchronously."""
        b, D = self.batch, self.dc.n_dof
        pin_t, pin_f = self._pinned()
        s = stream()
        s.synchronize()   # the previous run's copies out of the pinned buffers are done
        if isinstance(thetas, (list, tuple)):
            # one flat concatenate per array into the pinned buffers (about half the
            # time of np.stack over 1024 small rows)
            np.concatenate(thetas, out=pin_t.numpy().reshape(-1), casting="same_kind")
            fz = pin_f.numpy().reshape(-1)
            if all(getattr(f, "dtype", None) == np.bool_ for f in frozen):
                np.concatenate(frozen, out=fz.view(np.bool_))
            else:
                np.concatenate([np.asarray(f, np.uint8) for f in frozen], out=fz)
        else:
            pin_t.numpy()[...] = np.asarray(thetas, float)
            pin_f.numpy()[...] = np.asarray(frozen, np.uint8)
        with torch.cuda.stream(s):
            b.reset_status()
            _prep_clash_key(b)
            b.t["theta"][:, :D].copy_(pin_t, non_blocking=True)
            b.t["frozen"][:, :D].copy_(pin_f, non_blocking=True)

    def load_device(self, theta_dev):
        """theta already on the device ([B, D] float64)."""
        b, D = self.batch, self.dc.n_dof
        with torch.cuda.stream(stream()):
            b.reset_status()
            _prep_clash_key(b)
            b.t["theta"][:, :D].copy_(theta_dev)

    def prepare(self, n_iters: int):
        """Capture the graphs run_graph(n_iters) will replay (no launch)."""
        lib = N.lib()
        cs, fs, bs = N.ref(self.dc.struct), N.ref(self.df.struct_for(False)), N.ref(self.batch.struct)
        ss = N.ref(_step_struct(self.step))
        sizes = {min(self.chunk, n_iters)}
        if n_iters % self.chunk:
            sizes.add(n_iters % self.chunk)
        with torch.cuda.stream(stream()):
            for k in sizes:
                N.check(lib.kf_fold_graph_prepare(cs, fs, bs, ss, k, _sp()), "kf_fold_graph_prepare")

    def run_graph(self, n_iters: int):
        """Enqueue n_iters iterations (no host sync)."""
        lib = N.lib()
        cs, fs, bs = N.ref(self.dc.struct), N.ref(self.df.struct_for(False)), N.ref(self.batch.struct)
        ss = N.ref(_step_struct(self.step))
        left = n_iters
        while left > 0:
            k = min(self.chunk, left)
            N.check(lib.kf_fold_iterations(cs, fs, bs, ss, k, _sp()), "kf_fold_iterations")
            left -= k

    def run(self):
        with torch.cuda.stream(stream()):
            _run_loop(self.dc, self.df, self.batch, self.step, self.chunk)

    def result(self) -> EnsembleResult:
        b, D = self.batch, self.dc.n_dof
        with torch.cuda.stream(stream()):
            sa = b.status_array()
            bad = np.flatnonzero(sa["error"])
            if len(bad):
                k = int(bad[0])
                st = b.status()[k]
                _raise_status(st, self.df, b, prefix=f"trajectory {k}: aborted at iteration {st.err_iter}: ", b=k)
            iters = sa["iter"].astype(np.int64)
            K = int(iters.max()) if len(iters) else 0
            rec = b.t["rec_energy"][:, :max(K, 1)].cpu().numpy()[:, :K]
            th = b.t["theta"][:, :D].cpu().numpy()
            thetas = (b.t["rec_theta"][:, :K].cpu().numpy()
                      if b.t["rec_theta"] is not None else None)
        # record rows past a trajectory's own stop hold a previous run's values (the
        # record buffers are reused, not cleared): zero them
        past = np.arange(K)[None, :] >= iters[:, None]
        if past.any():
            rec[past] = 0.0
            if thetas is not None:
                thetas[past] = 0.0
        names = {code: N.REASONS.get(int(code), "max_iters") for code in np.unique(sa["reason"])}
        return EnsembleResult(theta=th, energies=rec, iterations=iters,
                              reasons=[names[r] for r in sa["reason"]],
                              thetas=thetas, n_pairs=sa["n_pairs"].astype(np.int64))


_runner_cache = _IdCache()


def fold_ensemble(chain, confs, fld, step, record_theta: bool = False) -> EnsembleResult:
    confs = list(confs)
    dc = device_chain(chain)
    df = device_field(fld, dc.n_atoms)
    # the device tables in the key: a re-uploaded chain or field (mutated arrays,
    # another pair precision) builds a new runner instead of reusing stale tables
    key = (len(confs), repr(step), bool(record_theta), id(fld), id(dc), id(df), pair_precision())
    runner = _runner_cache.get(chain, hash(key),
                               lambda: EnsembleRunner(chain, fld, len(confs), step, record_theta=record_theta))
    if runner.dc is not dc or runner.df is not df:
        runner = EnsembleRunner(chain, fld, len(confs), step, record_theta=record_theta)
    if runner.df.solvation and step.max_iters > 0:
        check_cav_cutoff(fld.params, fld.config.solvation_cfg, fld.config.cutoffs.cav)
    runner.load([c.theta for c in confs], [c.frozen for c in confs])
    runner.run()
    return runner.result()


def single_points(chain, thetas, fld) -> list:
    """Energy-only FK + field for a batch of conformations (kcm.py:358-360, :406-419)."""
    thetas = np.asarray(thetas, float)
    dc = device_chain(chain)
    df = device_field(fld, dc.n_atoms)
    if df.solvation:
        check_cav_cutoff(fld.params, fld.config.solvation_cfg, fld.config.cutoffs.cav)
    B = len(thetas)
    b = df.batch(dc, B)
    fs = df.struct_for(False)
    with torch.cuda.stream(stream()):
        b.reset_status()
        _prep_clash_key(b)
        b.t["theta"][:, :dc.n_dof].copy_(torch.from_numpy(thetas))
        _call("kf_fk", N.ref(dc.struct), N.ref(b.struct), _sp())
        _call("kf_nonbonded", N.ref(fs), N.ref(b.struct), _sp())
        if df.solvation:
            _call("kf_solvation", N.ref(fs), N.ref(b.struct), _sp())
        _call("kf_energy_reduce", N.ref(fs), N.ref(b.struct), dc.n_atoms, _sp())
        sts = b.status()
        for k, st in enumerate(sts):
            if st.error:
                _raise_status(st, df, b, b=k)
        e = b.t["energy"].cpu().numpy()
    return [EnergyBreakdown(float(x[0]), float(x[1]), float(x[2])) for x in e]


# --------------------------------------------------------------------------
# wrenches, torques, step (API)
# --------------------------------------------------------------------------

def link_wrenches(chain, positions, forces):
    dc = device_chain(chain)
    with torch.cuda.stream(stream()):
        p = _up(positions, np.float64)
        f = _up(forces, np.float64)
        w = torch.zeros(dc.n_links, 6, dtype=torch.float64, device=p.device)
        _call("kf_link_wrenches", N.ref(dc.struct), _p(p), _p(f), _p(w), _sp())
        out = w.cpu().numpy()
    return out[:, :3].copy(), out[:, 3:].copy()


def joint_torques(chain, state, wrenches) -> np.ndarray:
    dc = device_chain(chain)
    L = dc.n_links
    X = np.zeros((L, 16))
    for k in range(L):
        X[k, :9] = np.asarray(state.transforms[k], float).reshape(9)
        X[k, 9:12] = state.joint_points[k]
        if state.axes[k] is not None:
            X[k, 12:15] = state.axes[k]
    wr = np.concatenate([np.asarray(wrenches.force, float), np.asarray(wrenches.torque, float)], axis=1)
    with torch.cuda.stream(stream()):
        xt = _up(X, np.float64)
        wt = _up(wr, np.float64)
        dev = xt.device
        side = torch.zeros(max(dc.n_res, 1), 6, dtype=torch.float64, device=dev)
        suf = torch.zeros(max(dc.n_bb, 1), 6, dtype=torch.float64, device=dev)
        tau = torch.zeros(max(dc.n_dof, 1), dtype=torch.float64, device=dev)
        _call("kf_joint_torques", N.ref(dc.struct), _p(xt), _p(wt), _p(side), _p(suf), _p(tau), _sp())
        return tau[:dc.n_dof].cpu().numpy()


def kcm_step(tau, conf, kappa: float):
    D = len(tau)
    with torch.cuda.stream(stream()):
        t = _up(tau, np.float64)
        th = _up(conf.theta, np.float64)
        fr = _up(conf.frozen, np.uint8)
        out = torch.zeros(D, dtype=torch.float64, device=t.device)
        dl = torch.zeros(D, dtype=torch.float64, device=t.device)
        _call("kf_kcm_step", _p(t), _p(th), _p(fr), D, float(kappa), _p(out), _p(dl), _sp())
        theta_out, deltas = out.cpu().numpy(), dl.cpu().numpy()
    return theta_out, deltas, bool(np.any(deltas != 0.0))


# --------------------------------------------------------------------------
# spatial API (reference grid, tables, filtering)
# --------------------------------------------------------------------------

def build_grid(positions, config):
    from .spatial import HashGrid, reference_cell_edge
    pos = np.asarray(positions, float)
    if pos.ndim != 2 or pos.shape[1] != 3 or len(pos) < 1:
        raise ConfigurationError("positions must be a non-empty (n, 3) array")
    n = len(pos)
    with torch.cuda.stream(stream()):
        p = _up(pos, np.float64)
        dev = p.device
        mm = torch.zeros(7, dtype=torch.float64, device=dev)
        _call("kf_bbox", _p(p), n, _p(mm), _sp())
        mmh = mm.cpu().numpy()
        if mmh[6] > 0:
            raise ConfigurationError("non-finite coordinates cannot be hashed")
        r_min, r_max = mmh[0:3].copy(), mmh[3:6].copy()
        cell, dims = reference_cell_edge(r_min, r_max, n, config)
        n_keys = int(np.prod(dims))
        rmin_t = _up(r_min, np.float64)
        dims_t = _up(dims, np.int64)
        cells = torch.empty(n, 3, dtype=torch.int64, device=dev)
        lin = torch.empty(n, dtype=torch.int64, device=dev)
        _call("kf_grid_cells", _p(p), n, _p(rmin_t), float(cell), _p(dims_t), _p(cells), _p(lin), _sp())
        counts, starts, order = _counting_sort(lin, n, n_keys)
        scratch = torch.empty(n_keys + 1024, dtype=torch.int64, device=dev)
        dest = torch.empty(n_keys + 1, dtype=torch.int64, device=dev)
        occ = torch.empty(n_keys, dtype=torch.int64, device=dev)
        occ_st = torch.empty(n_keys + 1, dtype=torch.int64, device=dev)
        _call("kf_grid_occupied", _p(counts), _p(starts), n_keys, _p(scratch), _p(dest), _p(occ),
              _p(occ_st), _sp())
        n_occ = int(dest[n_keys].item())
        occupied = occ[:n_occ].cpu().numpy()
        st = np.append(occ_st[:n_occ].cpu().numpy(), n)
        cell_index = cells.cpu().numpy()
        atom_order = order.cpu().numpy()
    return HashGrid(cell_size=float(cell), r_min=r_min, r_max=r_max, dims=dims,
                    cell_index=cell_index, _occupied=occupied, _starts=st,
                    _atom_order=atom_order, positions=pos)


def _counting_sort(keys_t, n, n_keys):
    dev = keys_t.device
    counts = torch.empty(max(n_keys, 1), dtype=torch.int32, device=dev)
    starts = torch.empty(n_keys + 1, dtype=torch.int64, device=dev)
    order = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    scratch = torch.empty(n_keys + 1024, dtype=torch.int64, device=dev)
    _call("kf_counting_sort", _p(keys_t), n, n_keys, _p(counts), _p(starts), _p(order), _p(scratch), _sp())
    return counts, starts, order[:n]


def build_neighbor_table(grid, d_cut: float):
    from .spatial import NeighborTable, reference_stencil
    if d_cut <= 0:
        raise ConfigurationError("cutoff must be positive")
    n = int(len(grid._atom_order))
    dims = np.asarray(grid.dims, np.int64)
    offs = reference_stencil(grid.cell_size, d_cut)
    offs = offs[(np.abs(offs) < dims).all(axis=1)]
    n_keys = int(np.prod(dims))
    with torch.cuda.stream(stream()):
        ci = _up(grid.cell_index, np.int64)
        dev = ci.device
        dims_t = _up(dims, np.int64)
        lin = _up(grid.linear_ids(np.asarray(grid.cell_index, np.int64)), np.int64)
        _, starts, order = _counting_sort(lin, n, n_keys)
        sten = _up(offs, np.int32)
        row_len = torch.empty(n, dtype=torch.int64, device=dev)
        _call("kf_neighbor_rows_count", _p(ci), _p(dims_t), n, _p(starts), _p(sten), len(offs),
              _p(row_len), _sp())
        offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
        scratch = torch.empty(1024, dtype=torch.int64, device=dev)
        _call("kf_scan_exclusive_i64", _p(row_len), n, _p(offsets), _p(scratch), _sp())
        total = int(offsets[n].item())
        nbrs = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
        _call("kf_neighbor_rows_fill", _p(ci), _p(dims_t), n, _p(starts), _p(order), _p(sten), len(offs),
              _p(offsets), _p(nbrs), _sp())
        _call("kf_sort_rows", _p(offsets), n, _p(nbrs), _sp())
        return NeighborTable(d_cut=float(d_cut), offsets=offsets.cpu().numpy(),
                             neighbors=nbrs[:total].cpu().numpy())


def _filter(table, positions, d_cut, upper_only: bool):
    pos = np.asarray(positions, float)
    n = len(table.offsets) - 1
    offsets = np.asarray(table.offsets, np.int64)
    nbrs = np.asarray(table.neighbors, np.int64)
    m = len(nbrs)
    p = _up(pos, np.float64)
    dev = p.device
    off_t = _up(offsets, np.int64)
    nb_t = _up(nbrs if m else np.zeros(1, np.int64), np.int64)
    keep = torch.zeros(max(m, 1), dtype=torch.uint8, device=dev)
    d2 = torch.zeros(max(m, 1), dtype=torch.float64, device=dev)
    _call("kf_filter_table", _p(p), _p(off_t), _p(nb_t), n, m, float(d_cut) * float(d_cut),
          int(upper_only), _p(keep), _p(d2), _sp())
    dest = torch.empty(m + 1, dtype=torch.int64, device=dev)
    scratch = torch.empty(m + 1024, dtype=torch.int64, device=dev)
    oi = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
    oj = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
    od = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
    _call("kf_compact_pairs", _p(off_t), _p(nb_t), n, m, _p(keep), _p(d2), _p(dest), _p(scratch),
          _p(oi), _p(oj), _p(od), _sp())
    k = int(dest[m].item())
    return p, off_t, dest, oi[:k], oj[:k], od[:k], n


def _device_pairs(table, positions, d_cut):
    """(i, j, d) as device tensors, with the reference's clash guard."""
    p, _, _, i, j, d, n = _filter(table, positions, d_cut, True)
    if len(d):
        am = torch.empty(1, dtype=torch.int64, device=d.device)
        _call("kf_argmin_f64", _p(d), len(d), _p(am), _sp())
        k = int(am.item())
        dk = float(d[k].item())
        if dk < MIN_DISTANCE:
            raise StericClashError(f"atoms {int(i[k].item())} and {int(j[k].item())} closer than "
                                   f"{MIN_DISTANCE} A (d={dk:.3e})")
    return p, i, j, d, n


def filtered_pairs(table, positions, d_cut):
    with torch.cuda.stream(stream()):
        _, _, _, i, j, d, _ = _filter(table, positions, d_cut, True)
        return i.cpu().numpy(), j.cpu().numpy(), d.cpu().numpy()


def extract_pairs(positions, table, d_cut):
    with torch.cuda.stream(stream()):
        _, i, j, d, _ = _device_pairs(table, positions, d_cut)
        return i.cpu().numpy(), j.cpu().numpy(), d.cpu().numpy()


def filtered_lists(table, positions, d_cut) -> list:
    with torch.cuda.stream(stream()):
        _, off_t, dest, _, oj, _, n = _filter(table, positions, d_cut, False)
        rows = torch.empty(n + 1, dtype=torch.int64, device=oj.device)
        _call("kf_row_kept_offsets", _p(off_t), n, _p(dest), _p(rows), _sp())
        if len(oj):
            _call("kf_sort_rows", _p(rows), n, _p(oj), _sp())
        r = rows.cpu().numpy()
        vals = oj.cpu().numpy()
    return [vals[r[a]:r[a + 1]] for a in range(n)]


# --------------------------------------------------------------------------
# forcefield API
# --------------------------------------------------------------------------

def _param_tables(params, weights, dielectric, n):
    fp = _fingerprint(np.asarray(params.q, float), np.asarray(params.R, float),
                      np.asarray(params.eps, float), np.array([n])) ^ id(weights) ^ hash(repr(dielectric))
    key_obj = params
    return _tree_cache.get(key_obj, fp, lambda: ParamTables(params, weights, dielectric, n))


def table_term(positions, params, table, weights, d_cut, dielectric, kind: int, what: str):
    pos = np.asarray(positions, float)
    n = len(pos)
    pt = _param_tables(params, weights, dielectric, n)
    with torch.cuda.stream(stream()):
        p, i, j, d, _ = _device_pairs(table, pos, d_cut)
        m = len(d)
        dev = p.device
        if what == "energy":
            e = torch.zeros(max(m, 1), dtype=torch.float64, device=dev)
            _call("kf_pair_terms", N.ref(pt.struct), _p(p), n, _p(i), _p(j), _p(d), None, m, kind,
                  _p(e), None, None, _sp())
            part = torch.empty(1024, dtype=torch.float64, device=dev)
            out = torch.zeros(1, dtype=torch.float64, device=dev)
            _call("kf_sum_f64", _p(e), m, _p(part), _p(out), _sp())
            return float(out.item())
        forces = torch.zeros(n, 3, dtype=torch.float64, device=dev)
        _call("kf_pair_terms", N.ref(pt.struct), _p(p), n, _p(i), _p(j), _p(d), None, m, kind,
              None, None, _p(forces), _sp())
        return forces.cpu().numpy()


def pair_quantities(params, i, j, d, w, kind, dielectric):
    i = np.asarray(i, np.int64)
    m = len(i)
    n = len(params.q)
    from .topology import UniformWeights
    pt = _param_tables(params, UniformWeights(1.0), dielectric, n)
    with torch.cuda.stream(stream()):
        it, jt = _up(i if m else np.zeros(1), np.int64), _up(j if m else np.zeros(1), np.int64)
        dt = _up(d if m else np.ones(1), np.float64)
        wt = _up(w if m else np.zeros(1), np.float64)
        dev = it.device
        e = torch.zeros(max(m, 1), dtype=torch.float64, device=dev)
        mag = torch.zeros(max(m, 1), dtype=torch.float64, device=dev)
        dummy = torch.zeros(3, dtype=torch.float64, device=dev)
        _call("kf_pair_terms", N.ref(pt.struct), _p(dummy), n, _p(it), _p(jt), _p(dt), _p(wt), m, kind,
              _p(e), _p(mag), None, _sp())
        return e[:m].cpu().numpy(), mag[:m].cpu().numpy()


def accumulate_pair_forces(n, positions, i, j, d, mag) -> np.ndarray:
    m = len(np.asarray(d))
    with torch.cuda.stream(stream()):
        p = _up(positions, np.float64)
        out = torch.zeros(n, 3, dtype=torch.float64, device=p.device)
        if m:
            it, jt, dt, mt = _up(i, np.int64), _up(j, np.int64), _up(d, np.float64), _up(mag, np.float64)
            _call("kf_scatter_pair_forces", _p(p), int(n), _p(it), _p(jt), _p(dt), _p(mt), m, _p(out), _sp())
        return out.cpu().numpy()


def classify_pairs(tree, i, j) -> np.ndarray:
    from .topology import TreeWeights
    m = len(i)
    if m == 0:
        return np.zeros(0, np.int64)
    n = len(tree.parent)
    holder = TreeWeights(tree)
    fp = _fingerprint(np.asarray(tree.parent), np.asarray(tree.residue_of), np.asarray(tree.chain_mask))
    dummy = type("P", (), {})()
    dummy.q = dummy.R = dummy.eps = dummy.gamma = np.ones(n)
    pt = _tree_cache.get(tree, fp, lambda: ParamTables(dummy, holder, None, n))
    with torch.cuda.stream(stream()):
        it, jt = _up(i, np.int64), _up(j, np.int64)
        out = torch.empty(m, dtype=torch.int64, device=it.device)
        _call("kf_classify_pairs", N.ref(pt.struct), _p(it), _p(jt), m, _p(out), _sp())
        return out.cpu().numpy()


# --------------------------------------------------------------------------
# solvation API
# --------------------------------------------------------------------------

def _pow2_cap(longest: int) -> int:
    # staged neighbours per atom: a power of two (the in-block bitonic sort), <= 2048 (smem)
    return int(min(max(1, 1 << int(math.ceil(math.log2(max(longest, 1))))), 2048))


def _csr(neighbors, n):
    lens = np.array([len(x) for x in neighbors], np.int64)
    if len(lens) != n:
        raise ConfigurationError("one neighbour list per atom is required")
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    flat = (np.concatenate([np.asarray(x, np.int64) for x in neighbors])
            if off[-1] else np.zeros(1, np.int64))
    return off, flat, int(lens.max()) if n else 0


def sasa_pass(positions, params, neighbors, sphere, config):
    pos = np.asarray(positions, float)
    n, N_s = len(pos), sphere.n
    r_off = np.asarray(params.R, float) + config.probe_radius
    r_off2 = r_off * r_off
    off, flat, longest = _csr(neighbors, n)
    cap = _pow2_cap(longest)
    with torch.cuda.stream(stream()):
        p = _up(pos, np.float64)
        dev = p.device
        ro, ro2 = _up(r_off, np.float64), _up(r_off2, np.float64)
        sm = _up(sphere.points, np.float64)
        ot, ft = _up(off, np.int64), _up(flat, np.int64)
        gm = _up(params.gamma, np.float64)
        counts = torch.zeros(max(n, 1), N_s, dtype=torch.uint8, device=dev)
        crit = torch.full((max(n, 1), N_s), -1, dtype=torch.int32, device=dev)
        cov = torch.zeros(max(n, 1), dtype=torch.int64, device=dev)
        fe, ae, cv = (torch.zeros(max(n, 1), dtype=torch.float64, device=dev) for _ in range(3))
        ovf = torch.zeros(1, dtype=torch.int32, device=dev)
        _call("kf_sasa_pass", _p(p), n, _p(ro), _p(ro2), _p(sm), N_s, _p(ot), _p(ft), 1e-3, cap,
              _p(counts), _p(crit), _p(cov), _p(gm), 4.0 * math.pi, _p(fe), _p(ae), _p(cv), _p(ovf), _sp())
        if int(ovf.item()) > 0:
            raise NativeLibraryError(f"neighbour list of {int(ovf.item())} reachable atoms exceeds {cap}")
        part = torch.empty(1024, dtype=torch.float64, device=dev)
        g = torch.zeros(1, dtype=torch.float64, device=dev)
        _call("kf_sum_f64", _p(cv), n, _p(part), _p(g), _sp())
        res = SasaResult(fe[:n].cpu().numpy(), ae[:n].cpu().numpy(), float(g.item()))
        states = ExposureStates(counts[:n].cpu().numpy(), crit[:n].cpu().numpy())
    return res, states


def solvation_forces(positions, params, neighbors, sphere, states, config) -> np.ndarray:
    pos = np.asarray(positions, float)
    n, N_s = len(pos), sphere.n
    r_off = np.asarray(params.R, float) + config.probe_radius
    r_off2 = r_off * r_off
    w_int, quantum = force_quantum(params, r_off, N_s, config.delta_r)
    off, flat, longest = _csr(neighbors, n)
    cap = _pow2_cap(longest)
    with torch.cuda.stream(stream()):
        p = _up(pos, np.float64)
        dev = p.device
        acc = torch.zeros(max(n, 1), 3, dtype=torch.int64, device=dev)
        ovf = torch.zeros(1, dtype=torch.int32, device=dev)
        keep = [_up(r_off, np.float64), _up(r_off2, np.float64), _up(w_int, np.int64),
                _up(sphere.points, np.float64), _up(off, np.int64), _up(flat, np.int64),
                _up(states.counts, np.uint8), _up(states.critical, np.int32)]
        ro, ro2, wi, sm, ot, ft, cn, cr = keep
        _call("kf_solvation_forces", _p(p), n, _p(ro), _p(ro2), _p(wi), _p(sm), N_s, _p(ot), _p(ft),
              _p(cn), _p(cr), float(config.delta_r), float(config.delta_r) + 1e-3, cap, _p(acc), _p(ovf),
              _sp())
        if int(ovf.item()) > 0:
            raise NativeLibraryError(f"neighbour list of {int(ovf.item())} reachable atoms exceeds {cap}")
        out = torch.zeros(max(n, 1), 3, dtype=torch.float64, device=dev)
        _call("kf_fixed_to_f64", _p(acc), 3 * n, float(quantum), _p(out), _sp())
        return out[:n].cpu().numpy()
