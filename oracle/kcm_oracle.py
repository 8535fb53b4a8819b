"""CPU oracle of the KCM hot path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (/root/reference/pkg/src/
kinefold, the `kinefold` 0.1.0 package) for the per-iteration KCM loop, used
as the parity checker of the GPU path and as the timed CPU baseline.  Only
tests/, __graft_entry__.smoke() and bench.py's CPU legs may import it; the
product (paper_1712_05012_b200) never does and has no CPU fallback.

Pinning: tests/test_oracle_golden.py checks every function here against
golden vectors produced by the real reference (tests/golden/make_golden.py,
run in the build container where /root/reference exists), and
tests/test_oracle_reference.py re-checks against the live reference whenever
it is importable.  Where the reference's numpy expressions fix the bit-level
result (einsum order of d2, (d*d).sum(-1) coverage tests, bincount scatter
order, int64 fixed point, np.mod wrapping) the same expressions are used.

Inputs are plain objects with the reference's attribute names (a
``kinefold.Chain`` or ``paper_1712_05012_b200.Chain``; params with q, R, eps,
gamma; weights with tree + table or a uniform value).
"""

from __future__ import annotations

import math

import numpy as np

COULOMB_K = 332.06
MIN_DISTANCE = 1e-6
SQRT3 = float(np.sqrt(3.0))


class OracleError(Exception):
    """Raised where the reference raises (message text kept)."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


# ---- geometry / FK (chain.py:240-261, geometry.py:26-46) -------------------

def rodrigues(axis, deg):
    t = math.radians(deg)
    c, s = math.cos(t), math.sin(t)
    x, y, z = axis
    k = np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])
    return np.eye(3) + s * k + (1.0 - c) * (k @ k)


def wrap(theta):
    return np.mod(theta, 360.0)


def fk(chain, theta):
    """Sequential link walk: returns (M list, P list, U list, positions)."""
    links = chain.links
    M, P, U = [None] * len(links), [None] * len(links), [None] * len(links)
    pos = np.empty((len(chain.atom_names), 3))
    for li, ln in enumerate(links):
        if ln.kind == "ground":
            M[li], P[li] = np.eye(3), np.zeros(3)
        else:
            par = links[ln.parent]
            P[li] = P[ln.parent] + M[ln.parent] @ par.body0
            M[li] = M[ln.parent] @ rodrigues(ln.axis0, float(theta[ln.dof]))
            U[li] = M[li] @ ln.axis0
        idx = ln.atom_indices
        if idx.size:
            pos[idx] = P[li] + (chain.zp_pos[idx] - ln.point0) @ M[li].T
    return M, P, U, pos


# ---- spatial (spatial.py:83-259) ---------------------------------------------

def grid(positions, alpha=1.0, min_cell=1.0):
    positions = np.asarray(positions, float)
    if not np.isfinite(positions).all():
        raise OracleError("config", "non-finite coordinates cannot be hashed")
    n = len(positions)
    lo, hi = positions.min(axis=0), positions.max(axis=0)
    ext = hi - lo
    vol = float(np.prod(ext))
    cell = max((vol / (alpha * n)) ** (1.0 / 3.0) if vol > 0 else 0.0, min_cell)
    dims = np.maximum(np.ceil(ext / cell).astype(np.int64), 1)
    ci = np.floor((positions - lo) / cell).astype(np.int64)
    np.clip(ci, 0, dims - 1, out=ci)
    key = (ci[:, 0] * dims[1] + ci[:, 1]) * dims[2] + ci[:, 2]
    order = np.argsort(key, kind="stable")
    occ, first = np.unique(key[order], return_index=True)
    return dict(cell=float(cell), r_min=lo, r_max=hi, dims=dims, cell_index=ci,
                occupied=occ, starts=np.append(first, n), order=order)


def stencil(cell, d_cut):
    rc = d_cut + SQRT3 * cell
    r = int(np.floor(rc / cell))
    ax = np.arange(-r, r + 1)
    o = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), -1).reshape(-1, 3)
    return o[(o.astype(float) ** 2).sum(axis=1) * cell * cell <= rc * rc]


def neighbor_table(g, d_cut):
    """Superset rows: all atoms of stencil cells, ascending, self excluded."""
    dims = g["dims"]
    offs = stencil(g["cell"], d_cut)
    offs = offs[(np.abs(offs) < dims).all(axis=1)]
    where = {int(k): (int(g["starts"][t]), int(g["starts"][t + 1]))
             for t, k in enumerate(g["occupied"])}
    n = len(g["order"])
    rows = [None] * n
    for t, k in enumerate(g["occupied"]):
        c = np.array([k // (dims[1] * dims[2]), (k // dims[2]) % dims[1], k % dims[2]])
        nb = c + offs
        ok = ((nb >= 0) & (nb < dims)).all(axis=1)
        lin = (nb[ok, 0] * dims[1] + nb[ok, 1]) * dims[2] + nb[ok, 2]
        parts = [g["order"][slice(*where[int(x)])] for x in lin if int(x) in where]
        members = np.sort(np.concatenate(parts)) if parts else np.zeros(0, np.int64)
        for a in g["order"][g["starts"][t]:g["starts"][t + 1]]:
            rows[a] = members[members != a]
    lens = np.array([len(r) for r in rows], np.int64)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    flat = np.concatenate(rows).astype(np.int64) if n else np.zeros(0, np.int64)
    return off, flat


def table_pairs(off, flat, positions, d_cut):
    n = len(off) - 1
    i = np.repeat(np.arange(n), np.diff(off))
    up = flat > i
    i, j = i[up], flat[up]
    diff = positions[i] - positions[j]
    d2 = np.einsum("ij,ij->i", diff, diff)
    k = d2 <= d_cut * d_cut
    return i[k], j[k], np.sqrt(d2[k])


def table_lists(off, flat, positions, d_cut):
    n = len(off) - 1
    i = np.repeat(np.arange(n), np.diff(off))
    diff = positions[i] - positions[flat]
    d2 = np.einsum("ij,ij->i", diff, diff)
    k = d2 <= d_cut * d_cut
    i, j = i[k], flat[k]
    b = np.searchsorted(i, np.arange(n + 1))
    return [np.sort(j[b[a]:b[a + 1]]) for a in range(n)]


def pairs(positions, d_cut, alpha=1.0):
    g = grid(positions, alpha)
    off, flat = neighbor_table(g, d_cut)
    return table_pairs(off, flat, np.asarray(positions, float), d_cut)


# ---- classification (topology.py:153-195) -----------------------------------

def classes(tree, i, j):
    p, gp, gg = tree.parent, tree.grandparent, tree.greatgrand
    eq = lambda a, b: (a == b) & (a >= 0)  # noqa: E731
    out = np.full(len(i), 4, np.int64)
    near = tree.chain_mask[i] & tree.chain_mask[j] & (np.abs(tree.residue_of[i] - tree.residue_of[j]) <= 1)
    a, b = i[near], j[near]
    c = np.full(len(a), 4, np.int64)
    c[eq(gg[a], b) | eq(gg[b], a) | eq(gp[a], p[b]) | eq(gp[b], p[a])] = 3
    c[eq(gp[a], b) | eq(gp[b], a) | eq(p[a], p[b])] = 2
    c[eq(p[a], b) | eq(p[b], a)] = 1
    out[near] = c
    return out


def pair_weights(weights, i, j, kind):
    if hasattr(weights, "tree"):
        t = weights.table
        tab = np.array([np.nan, 0.0, t.w13_elec, t.w14_elec, 1.0]) if kind == "elec" else \
            np.array([np.nan, 0.0, t.w13_vdw, t.w14_vdw, 1.0])
        return tab[classes(weights.tree, i, j)]
    return np.full(len(i), float(weights.value))


# ---- elec / vdW (forcefield.py:81-172) -----------------------------------------

def scatter(n, positions, i, j, d, mag):
    out = np.zeros((n, 3))
    if len(d) == 0:
        return out
    f = mag[:, None] * ((positions[i] - positions[j]) / d[:, None])
    for ax in range(3):
        out[:, ax] += np.bincount(i, weights=f[:, ax], minlength=n)
        out[:, ax] -= np.bincount(j, weights=f[:, ax], minlength=n)
    return out


def elec_terms(params, i, j, d, w, dielectric_mode="distance", kappa=1.0):
    kap = d if dielectric_mode == "distance" else np.full(len(d), kappa)
    num = COULOMB_K * w * params.q[i] * params.q[j]
    return num / (kap * d), num / (kap * d * d)


def vdw_terms(params, i, j, d, w):
    eps = np.sqrt(params.eps[i] * params.eps[j])
    dd = params.R[i] + params.R[j]
    r6 = dd**6 / d**6
    return w * eps * (r6 * r6 - 2.0 * r6), 12.0 * w * eps * (dd**12 / d**13 - dd**6 / d**7)


def clash_guard(i, j, d):
    if len(d) and float(d.min()) < MIN_DISTANCE:
        k = int(np.argmin(d))
        raise OracleError("clash", f"atoms {i[k]} and {j[k]} closer than {MIN_DISTANCE} A (d={d[k]:.3e})")


# ---- solvation (solvation.py:64-255) -------------------------------------------

def force_quantum(gamma, r_off, nq, dr):
    delta = 4.0 * math.pi * gamma * r_off * r_off / (nq * dr)
    peak = float(np.max(np.abs(delta))) if len(delta) else 0.0
    if peak == 0.0:
        return np.zeros(len(delta), np.int64), 1.0
    q = 2.0 ** (math.floor(math.log2(peak)) - 36)
    return np.round(delta / q).astype(np.int64), q


def sasa(positions, params, lists, points, probe=1.4):
    """Exposure counts (clamped at 2), critical coverer, f_exp, a_exp, g_cav."""
    positions = np.asarray(positions, float)
    n, nq = len(positions), len(points)
    ro = params.R + probe
    ro2 = ro * ro
    counts = np.zeros((n, nq), np.uint8)
    crit = np.full((n, nq), -1, np.int32)
    covered = np.zeros(n, np.int64)
    for a in range(n):
        nb = lists[a]
        if len(nb) == 0:
            continue
        pts = positions[a] + ro[a] * points
        diff = pts[:, None, :] - positions[nb][None, :, :]
        cov = (diff * diff).sum(-1) <= ro2[nb][None, :]
        c = np.minimum(cov.sum(1), 2)
        counts[a] = c
        one = c == 1
        if one.any():
            crit[a, one] = nb[np.argmax(cov[one], axis=1)]
        covered[a] = int((c > 0).sum())
    f_exp = (nq - covered) / float(nq)
    a_exp = f_exp * (4.0 * math.pi * ro2)
    return counts, crit, f_exp, a_exp, float(np.sum(params.gamma * a_exp))


def solvation_acc(positions, params, lists, points, counts, crit, probe=1.4, dr=1e-2):
    """int64 fixed-point forward-difference accumulator and its quantum."""
    positions = np.asarray(positions, float)
    n, nq = len(positions), len(points)
    ro = params.R + probe
    ro2 = ro * ro
    w, quantum = force_quantum(params.gamma, ro, nq, dr)
    acc = np.zeros((n, 3), np.int64)
    for a in range(n):
        nb = lists[a]
        if w[a] == 0 or len(nb) == 0:
            continue
        pts = positions[a] + ro[a] * points
        e0 = np.flatnonzero(counts[a] == 0)
        e1 = np.flatnonzero(counts[a] == 1)
        for s in range(3):
            if e0.size:
                moved = positions[nb].copy()
                moved[:, s] += dr
                diff = pts[e0][:, None, :] - moved[None, :, :]
                hits = ((diff * diff).sum(-1) <= ro2[nb][None, :]).sum(0)
                tot = int(hits.sum())
                if tot:
                    acc[a, s] -= tot * w[a]
                    pos_hits = hits > 0
                    np.add.at(acc[:, s], nb[pos_hits], hits[pos_hits] * w[a])
            if e1.size:
                jo = crit[a, e1]
                moved = positions[jo]
                moved[:, s] += dr
                dd = pts[e1] - moved
                freed = (dd * dd).sum(-1) > ro2[jo]
                if freed.any():
                    acc[a, s] += int(freed.sum()) * w[a]
                    np.subtract.at(acc[:, s], jo[freed], w[a])
    return acc, quantum


def sample_sphere(n):
    n_orb = max(2 * int(round(math.sqrt(math.pi * n) / 4.0)), 2)
    polar = (np.arange(n_orb) + 0.5) * math.pi / n_orb
    wt = np.sin(polar)
    ideal = n * wt / wt.sum()
    cnt = np.floor(ideal).astype(int)
    cnt[np.argsort(-(ideal - cnt), kind="stable")[:n - cnt.sum()]] += 1
    out = np.empty((n, 3))
    at = 0
    for t, c in enumerate(cnt):
        if c == 0:
            continue
        az = 2.0 * math.pi * (np.arange(c) + (t * 0.618033988749895) % 1.0) / c
        s, z = math.sin(polar[t]), math.cos(polar[t])
        out[at:at + c] = np.stack([s * np.cos(az), s * np.sin(az), np.full(c, z)], 1)
        at += c
    return out / np.linalg.norm(out, axis=1, keepdims=True)


# ---- one field evaluation (kcm.py:104-150) ----------------------------------------

class OracleField:
    def __init__(self, params, weights, cut_elec=9.0, cut_vdw=5.0, cut_cav=8.0, solvation=False,
                 dielectric_mode="distance", kappa=1.0, alpha=1.0, samples=1024, probe=1.4, dr=1e-2):
        self.params, self.weights = params, weights
        self.ce, self.cv, self.cc = cut_elec, cut_vdw, cut_cav
        self.solvation, self.mode, self.kappa, self.alpha = solvation, dielectric_mode, kappa, alpha
        self.points = sample_sphere(samples) if solvation else None
        self.probe, self.dr = probe, dr

    def evaluate(self, positions):
        positions = np.asarray(positions, float)
        n = len(positions)
        act = max(self.ce, self.cv, self.cc) if self.solvation else max(self.ce, self.cv)
        g = grid(positions, self.alpha)
        off, flat = neighbor_table(g, act)
        i, j, d = table_pairs(off, flat, positions, max(self.ce, self.cv))
        clash_guard(i, j, d)
        ke, kv = d <= self.ce, d <= self.cv
        ee, me = elec_terms(self.params, i[ke], j[ke], d[ke], pair_weights(self.weights, i[ke], j[ke], "elec"),
                            self.mode, self.kappa)
        ev, mv = vdw_terms(self.params, i[kv], j[kv], d[kv], pair_weights(self.weights, i[kv], j[kv], "vdw"))
        forces = np.zeros((n, 3))
        forces += scatter(n, positions, i[ke], j[ke], d[ke], me)
        forces += scatter(n, positions, i[kv], j[kv], d[kv], mv)
        g_cav, extra = 0.0, {}
        if self.solvation:
            need = 2.0 * (float(np.max(self.params.R)) + self.probe)
            if need > self.cc:
                raise OracleError("config", f"cavity cutoff {self.cc} A below 2(R_max + probe) = {need:.2f} A")
            lists = table_lists(off, flat, positions, self.cc)
            counts, crit, f_exp, a_exp, g_cav = sasa(positions, self.params, lists, self.points, self.probe)
            acc, q = solvation_acc(positions, self.params, lists, self.points, counts, crit, self.probe, self.dr)
            forces += acc.astype(float) * q
            extra = dict(counts=counts, critical=crit, f_exp=f_exp, a_exp=a_exp, acc=acc, quantum=q)
        energies = (float(ee.sum()), float(ev.sum()), g_cav)
        return forces, energies, dict(i=i, j=j, d=d, **extra)


# ---- wrenches, torques, step, loop (kcm.py:177-351) ---------------------------------

def wrenches(chain, positions, forces):
    L = len(chain.links)
    mom = np.cross(positions, forces)
    F = np.stack([np.bincount(chain.atom_link, weights=forces[:, a], minlength=L) for a in range(3)], 1)
    T = np.stack([np.bincount(chain.atom_link, weights=mom[:, a], minlength=L) for a in range(3)], 1)
    return F, T


def torques(chain, U, P, F, T):
    links = chain.links
    tau = np.zeros(len(links) - 1)
    proj = lambda li, f, t: float(U[li] @ t - np.cross(U[li], P[li]) @ f)  # noqa: E731
    m = chain.n_residues
    side_f, side_t = np.zeros((m, 3)), np.zeros((m, 3))
    per_res = {}
    for li, ln in enumerate(links):
        if ln.kind == "chi":
            per_res.setdefault(ln.residue, []).append(li)
    for r, lis in per_res.items():
        f, t = np.zeros(3), np.zeros(3)
        for li in sorted(lis, key=lambda x: links[x].chi_index)[::-1]:
            f, t = f + F[li], t + T[li]
            tau[links[li].dof] = proj(li, f, t)
        side_f[r], side_t[r] = f, t
    f, t = np.zeros(3), np.zeros(3)
    bb = sorted((li for li, ln in enumerate(links) if ln.kind in ("phi", "psi")), key=lambda x: links[x].dof)
    for li in bb[::-1]:
        f, t = f + F[li], t + T[li]
        if links[li].kind == "phi":
            f, t = f + side_f[links[li].residue], t + side_t[links[li].residue]
        tau[links[li].dof] = proj(li, f, t)
    return tau


def step(tau, theta, frozen, kappa):
    free = ~np.asarray(frozen, bool)
    if not free.any():
        raise OracleError("config", "cannot step with every joint frozen")
    tmax = float(np.max(np.abs(tau[free])))
    if tmax == 0.0:
        return theta.copy(), np.zeros_like(tau)
    delta = np.where(free, kappa * tau / tmax, 0.0)
    return wrap(wrap(theta + np.where(frozen, 0.0, delta))), delta


def fold(chain, theta, frozen, fld: OracleField, kappa=0.5, max_iters=2000, torque_tol=0.0,
         torque_tol_rel=1e-4, energy_window=20, energy_tol=0.02):
    """Returns dict(energies [K,3], tau_max [K], thetas [K,D], final, reason)."""
    theta = wrap(np.asarray(theta, float))
    frozen = np.asarray(frozen, bool)
    E, tm, th = [], [], []
    tau0, reason = None, "max_iters"
    for it in range(max_iters):
        M, P, U, pos = fk(chain, theta)
        try:
            forces, e, _ = fld.evaluate(pos)
        except OracleError as exc:
            raise OracleError(exc.kind, f"aborted at iteration {it}: {exc}") from exc
        F, T = wrenches(chain, pos, forces)
        tau = torques(chain, U, P, F, T)
        free = ~frozen
        tmax = float(np.max(np.abs(tau[free]))) if free.any() else 0.0
        E.append(e), tm.append(tmax), th.append(theta.copy())
        if tau0 is None:
            tau0 = tmax
        if tmax == 0.0:
            reason = "torque-free"
            break
        if torque_tol > 0 and tmax < torque_tol:
            reason = "torque tolerance"
            break
        if torque_tol_rel > 0 and tmax < torque_tol_rel * tau0:
            reason = "torque tolerance (relative)"
            break
        if energy_window and it >= energy_window:
            g = lambda k: E[k][0] + E[k][1] + E[k][2]  # noqa: E731
            if abs(g(it) - g(it - energy_window)) < energy_tol:
                reason = "energy plateau"
                break
        theta, _ = step(tau, theta, frozen, kappa)
    return dict(energies=np.array(E).reshape(-1, 3), tau_max=np.array(tm), thetas=np.array(th),
                final=theta, reason=reason)


def einsum_order_selftest() -> str:
    """Which association np.einsum('ij,ij->i') uses on this host."""
    rng = np.random.default_rng(7)
    d = rng.normal(size=(200000, 3)) * 5
    e = np.einsum("ij,ij->i", d, d)
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    for name, v in (("(xx+zz)+yy", (x * x + z * z) + y * y), ("(xx+yy)+zz", (x * x + y * y) + z * z),
                    ("(yy+zz)+xx", (y * y + z * z) + x * x)):
        if np.array_equal(v, e):
            return name
    return "other"
