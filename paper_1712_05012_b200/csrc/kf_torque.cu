// Link wrenches, suffix-scan joint torques, energy reduction, records, stop
// tests and the max-normalised compliance step (K6 + K7).
//
// Reference: link_wrenches (/root/reference/pkg/src/kinefold/kcm.py:177-188),
// joint_torques (:196-240), kcm_step (:264-274) with apply_deltas
// (chain.py:93-101), and fold's per-iteration bookkeeping (kcm.py:325-350).
//
// Wrenches repeat the reference's arithmetic (numpy cross product, bincount
// summation in ascending atom order), so they are bit-identical given the
// same positions and forces.  Joint torques replace the sequential suffix
// loop with a blocked parallel suffix scan of 6-vectors (one CTA per
// trajectory); tau_max is an exact max-reduction and the step reproduces
// numpy's float remainder twice, so theta' is bit-identical given tau.
#include "kf_common.cuh"
#ifdef TQ_TIMING
#include <cstdio>
#endif

namespace {

constexpr int TQ_THREADS = 512;

struct W6 { double f[3], t[3]; };

KF_DEV W6 w6_zero() { W6 r; for (int k = 0; k < 3; ++k) r.f[k] = r.t[k] = 0.0; return r; }
KF_DEV W6 w6_load(const double *s) { W6 r; for (int k = 0; k < 3; ++k) { r.f[k] = s[k]; r.t[k] = s[3 + k]; } return r; }
KF_DEV void w6_store(double *d, const W6 &r) { for (int k = 0; k < 3; ++k) { d[k] = r.f[k]; d[3 + k] = r.t[k]; } }
KF_DEV void w6_add(W6 &a, const W6 &b) { for (int k = 0; k < 3; ++k) { a.f[k] += b.f[k]; a.t[k] += b.t[k]; } }

// tau = u . T - (u x p) . F  (kcm.py:204-207), u = current axis, p = joint point
KF_DEV double project(const double *X, const W6 &w) {
    const double u0 = X[12], u1 = X[13], u2 = X[14];
    const double p0 = X[9], p1 = X[10], p2 = X[11];
    const double c0 = u1 * p2 - u2 * p1, c1 = u2 * p0 - u0 * p2, c2 = u0 * p1 - u1 * p0;
    return (u0 * w.t[0] + u1 * w.t[1] + u2 * w.t[2]) - (c0 * w.f[0] + c1 * w.f[1] + c2 * w.f[2]);
}

// F_l = sum F_a, T_l = sum r_a x F_a over the link's atoms in ascending order
// (np.cross + np.bincount, kcm.py:181-187): exact same roundings.
// One link's wrench: F = sum F_a, T = sum r_a x F_a over its atoms in ascending
// order (np.cross + np.bincount, kcm.py:181-187): exact same roundings.
KF_DEV void link_wrench(const kf_chain_t &c, int l, const double *pos, const double *frc, double *o) {
    double F0 = 0.0, F1 = 0.0, F2 = 0.0, T0 = 0.0, T1 = 0.0, T2 = 0.0;
    for (int e = c.link_atom_off[l]; e < c.link_atom_off[l + 1]; ++e) {
        const int a = c.link_atoms[e];
        const double r0 = pos[3 * a], r1 = pos[3 * a + 1], r2 = pos[3 * a + 2];
        const double g0 = frc[3 * a], g1 = frc[3 * a + 1], g2 = frc[3 * a + 2];
        F0 = xadd(F0, g0); F1 = xadd(F1, g1); F2 = xadd(F2, g2);
        T0 = xadd(T0, xsub(xmul(r1, g2), xmul(r2, g1)));
        T1 = xadd(T1, xsub(xmul(r2, g0), xmul(r0, g2)));
        T2 = xadd(T2, xsub(xmul(r0, g1), xmul(r1, g0)));
    }
    o[0] = F0; o[1] = F1; o[2] = F2; o[3] = T0; o[4] = T1; o[5] = T2;
}

// Wrench of link l with every load issued before the sums: the first 4 atoms
// (the synthetic chains have <= 4 per link) come in one round of independent
// loads instead of a dependent chain per atom.  Same arithmetic and order as
// link_wrench.
KF_DEV void link_wrench_pf(const kf_chain_t &c, int l, const double *__restrict__ pos,
                           const double *__restrict__ frc, double *o) {
    constexpr int P = 4;
    const int e0 = c.link_atom_off[l], e1 = c.link_atom_off[l + 1];
    int a[P];
    double r[P][3], g[P][3];
#pragma unroll
    for (int u = 0; u < P; ++u) a[u] = e0 + u < e1 ? c.link_atoms[e0 + u] : -1;
#pragma unroll
    for (int u = 0; u < P; ++u)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            r[u][q] = a[u] >= 0 ? pos[3 * a[u] + q] : 0.0;
            g[u][q] = a[u] >= 0 ? frc[3 * a[u] + q] : 0.0;
        }
    double F0 = 0.0, F1 = 0.0, F2 = 0.0, T0 = 0.0, T1 = 0.0, T2 = 0.0;
#pragma unroll
    for (int u = 0; u < P; ++u) {
        if (a[u] < 0) break;
        F0 = xadd(F0, g[u][0]); F1 = xadd(F1, g[u][1]); F2 = xadd(F2, g[u][2]);
        T0 = xadd(T0, xsub(xmul(r[u][1], g[u][2]), xmul(r[u][2], g[u][1])));
        T1 = xadd(T1, xsub(xmul(r[u][2], g[u][0]), xmul(r[u][0], g[u][2])));
        T2 = xadd(T2, xsub(xmul(r[u][0], g[u][1]), xmul(r[u][1], g[u][0])));
    }
    for (int e = e0 + P; e < e1; ++e) {   // links with more atoms: the rest in order
        const int at = c.link_atoms[e];
        const double r0 = pos[3 * at], r1 = pos[3 * at + 1], r2 = pos[3 * at + 2];
        const double g0 = frc[3 * at], g1 = frc[3 * at + 1], g2 = frc[3 * at + 2];
        F0 = xadd(F0, g0); F1 = xadd(F1, g1); F2 = xadd(F2, g2);
        T0 = xadd(T0, xsub(xmul(r1, g2), xmul(r2, g1)));
        T1 = xadd(T1, xsub(xmul(r2, g0), xmul(r0, g2)));
        T2 = xadd(T2, xsub(xmul(r0, g1), xmul(r1, g0)));
    }
    o[0] = F0; o[1] = F1; o[2] = F2; o[3] = T0; o[4] = T1; o[5] = T2;
}

__global__ void wrench_kernel(kf_chain_t c, int B, const double *__restrict__ pos_all,
                              const double *__restrict__ f_all, double *__restrict__ wrench_all,
                              const kf_status_t *status) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int L = c.n_links, n = c.n_atoms;
    if (gid >= (long long)B * L) return;
    const int b = (int)(gid / L), l = (int)(gid % L);
    if (status && (status[b].done || status[b].error)) return;
    link_wrench(c, l, pos_all + (size_t)b * n * 3, f_all + (size_t)b * n * 3, wrench_all + 6 * gid);
}

// Step 5 of a fold iteration (thread 0): energies, record, stop tests
// (kcm.py:325-350).  Returns the stop reason (KF_REASON_NONE: step).
KF_DEV int decide_iteration(const kf_batch_t &w, const kf_step_t &step, int b, int it, double tmax, double ge,
                            double gv, double gc, double sp, double sp5) {
    kf_status_t *st = w.status + b;
    double *e = w.energy + 3 * (size_t)b;
    e[0] = ge; e[1] = gv; e[2] = gc;
    st->n_pairs = (long long)(0.5 * sp);
    st->n_pairs_vdw = (long long)(0.5 * sp5);
    if (it < w.max_records) {
        double *rec = w.rec_energy + ((size_t)b * w.max_records + it) * 4;
        rec[0] = ge; rec[1] = gv; rec[2] = gc; rec[3] = tmax;
    }
    if (it == 0) st->tau0 = tmax;
    const double tau0 = st->tau0;
    int reason = KF_REASON_NONE;
    if (tmax == 0.0) reason = KF_REASON_TORQUE_FREE;
    else if (step.torque_tol > 0 && tmax < step.torque_tol) reason = KF_REASON_TORQUE_TOL;
    else if (step.torque_tol_rel > 0 && tmax < step.torque_tol_rel * tau0) reason = KF_REASON_TORQUE_TOL_REL;
    else if (step.energy_window && it >= step.energy_window && it < w.max_records) {
        const double *r0 = w.rec_energy + ((size_t)b * w.max_records + it) * 4;
        const double *r1 = w.rec_energy + ((size_t)b * w.max_records + it - step.energy_window) * 4;
        const double g0 = (r0[0] + r0[1]) + r0[2], g1 = (r1[0] + r1[1]) + r1[2];
        if (fabs(g0 - g1) < step.energy_tol) reason = KF_REASON_PLATEAU;
    }
    return reason;
}

// Step 6 over dofs [d0, d1) (the calling threads): theta record, then the
// compliance step theta' = mod(mod(theta + kappa*tau/tau_max)) on free joints.
KF_DEV void step_dofs(const kf_batch_t &w, const kf_step_t &step, int b, int D, int it, int reason,
                      const double *tau, double tmax, int d0, int d1, int tid, int nthreads) {
    const uint8_t *frozen = w.frozen + (size_t)b * D;
    double *th = w.theta + (size_t)b * D;
    if (w.record_theta && it < w.max_records) {
        double *rt = w.rec_theta + ((size_t)b * w.max_records + it) * D;
        for (int d = d0 + tid; d < d1; d += nthreads) rt[d] = th[d];
    }
    if (reason == KF_REASON_NONE)
        for (int d = d0 + tid; d < d1; d += nthreads) {
            const double delta = frozen[d] ? 0.0 : __ddiv_rn(xmul(step.kappa, tau[d]), tmax);
            th[d] = np_mod360(np_mod360(xadd(th[d], delta)));
        }
}

// Iteration counter and stop flags after the step (thread 0).
KF_DEV void close_iteration(kf_status_t *st, const kf_step_t &step, int it, int reason) {
    st->iter = it + 1;
    if (reason != KF_REASON_NONE) { st->done = 1; st->reason = reason; }
    else if (it + 1 >= step.max_iters) { st->done = 1; st->reason = KF_REASON_MAX_ITERS; }
}

// Steps 5-6 of a fold iteration by one CTA.
KF_DEV void finish_iteration(const kf_chain_t &c, const kf_batch_t &w, const kf_step_t &step, int b,
                             const double *tau, double tmax, double ge, double gv, double gc, double sp,
                             double sp5, int *stop_reason) {
    kf_status_t *st = w.status + b;
    const int it = st->iter;
    if (threadIdx.x == 0) *stop_reason = decide_iteration(w, step, b, it, tmax, ge, gv, gc, sp, sp5);
    __syncthreads();
    const int reason = *stop_reason;
    step_dofs(w, step, b, c.n_dof, it, reason, tau, tmax, 0, c.n_dof, threadIdx.x, blockDim.x);
    __syncthreads();
    if (threadIdx.x == 0) close_iteration(st, step, it, reason);
}

// Block-wide suffix scan of the threads' 6-vectors (later threads first):
// warp-level by shuffles, then the later warps' totals (wtot, one row per
// warp) added in a fixed order.  Returns the thread's exclusive suffix (the sum
// over later threads) and, in total, the block's sum.  Two block barriers.
KF_DEV W6 w6_block_suffix(const W6 &acc, double (*wtot)[6], W6 &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double v[6] = {acc.f[0], acc.f[1], acc.f[2], acc.t[0], acc.t[1], acc.t[2]};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        double u[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) u[q] = __shfl_down_sync(0xffffffffu, v[q], o);
        if (lane + o < 32)
#pragma unroll
            for (int q = 0; q < 6; ++q) v[q] += u[q];
    }
    __syncthreads();
    if (lane == 0)
        for (int q = 0; q < 6; ++q) wtot[wid][q] = v[q];
    __syncthreads();
    double tail[6] = {0, 0, 0, 0, 0, 0};   // totals of the later warps, last first
    for (int w2 = nw - 1; w2 > wid; --w2)
        for (int q = 0; q < 6; ++q) tail[q] += wtot[w2][q];
    double ex[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        const double nx = __shfl_down_sync(0xffffffffu, v[q], 1);
        ex[q] = lane < 31 ? nx + tail[q] : tail[q];
    }
    double all[6] = {0, 0, 0, 0, 0, 0};
    for (int w2 = nw - 1; w2 >= 0; --w2)
        for (int q = 0; q < 6; ++q) all[q] += wtot[w2][q];
    W6 later;
    for (int q = 0; q < 3; ++q) {
        later.f[q] = ex[q]; later.t[q] = ex[3 + q];
        total.f[q] = all[q]; total.t[q] = all[3 + q];
    }
    return later;
}

struct TorqueArgs {
    const double *link_T;      // [B][L][KF_XF_STRIDE]
    const double *wrench;      // [B][L][6]
    double *side_tot;          // [B][n_res][6]
    double *bb_suffix;         // [B][n_bb][6]
    double *tau;               // [B][D]
};

// One CTA per trajectory.  mode: 0 = torques only (API), 1 = fold iteration,
// 2 = energy reduction only (Field.evaluate)
// Torques (+ record, stop tests and step when mode == 1) of trajectory b by one CTA
// of NT threads; wsm: L x 6 doubles of shared memory for the fused wrenches.  Also
// the last phase of the fused fold iteration (kf_cluster.cu).
template <int NT>
KF_DEV void torque_step_cta(const kf_chain_t &c, const kf_field_t &f, const TorqueArgs &ta, const kf_batch_t &w,
                            const kf_step_t &step, int mode, int fuse_wrench, int e_first, int b, double *wsm) {
    kf_status_t *st = w.status ? w.status + b : nullptr;
    if (st && st->done) return;
    __shared__ double chunk[NT / 32][6];   // warp totals of the suffix scan
    __shared__ int stop_reason;
    if (st && st->error) {   // domain error this iteration: freeze, no record, no step
        if (threadIdx.x == 0) st->done = 1;
        return;
    }
    const int L = c.n_links, D = c.n_dof, R = c.n_res, nb = c.n_bb;
    const double *T = ta.link_T + (size_t)b * L * KF_XF_STRIDE;
    const double *Wr = ta.wrench + (size_t)b * L * 6;
#ifdef TQ_TIMING   // phase clocks of CTA 0 (measurement builds only)
    long long tk[8];
#define TQT(k) do { if (b == 0 && threadIdx.x == 0) tk[k] = clock64(); } while (0)
#else
#define TQT(k) do { } while (0)
#endif
    TQT(0);
    if (fuse_wrench) {   // wrenches of this iteration straight into shared memory
        const int n = c.n_atoms;
        for (int l = threadIdx.x; l < L; l += blockDim.x)
            link_wrench_pf(c, l, w.pos + (size_t)b * n * 3, w.forces + (size_t)b * n * 3, wsm + 6 * l);
        __syncthreads();
        Wr = wsm;
    }
    TQT(1);
    double *side = ta.side_tot + (size_t)b * R * 6;
    double *suf = ta.bb_suffix + (size_t)b * nb * 6;
    double *tau = ta.tau + (size_t)b * D;

    if (mode != 2) {
    // 1. side branches: plain suffix in chi order, total folded into phi (kcm.py:209-225)
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
        W6 agg = w6_zero();
        for (int e = c.chi_res_off[r + 1] - 1; e >= c.chi_res_off[r]; --e) {
            const int l = c.chi_links[e];
            w6_add(agg, w6_load(Wr + 6 * l));
            tau[c.link_dof[l]] = project(T + KF_XF_STRIDE * l, agg);
        }
        w6_store(side + 6 * r, agg);
    }
    __syncthreads();

    TQT(2);
    // 2. backbone reverse suffix over links in dof order (kcm.py:227-239)
    const int per = (nb + blockDim.x - 1) / blockDim.x;
    const int lo = min(nb, (int)threadIdx.x * per), hi = min(nb, lo + per);
    W6 acc = w6_zero();
    for (int k = hi - 1; k >= lo; --k) {
        w6_add(acc, w6_load(Wr + 6 * c.bb_by_dof[k]));
        const int r = c.bb_side_res[k];          // phi link: its residue's side total joins here
        if (r >= 0) w6_add(acc, w6_load(side + 6 * r));
        w6_store(suf + 6 * k, acc);
    }
    W6 total_unused;
    const W6 later = w6_block_suffix(acc, chunk, total_unused);
    for (int k = lo; k < hi; ++k) {
        const int l = c.bb_by_dof[k];
        W6 s = w6_load(suf + 6 * k);
        w6_add(s, later);
        tau[c.link_dof[l]] = project(T + KF_XF_STRIDE * l, s);
    }
    __syncthreads();
    }
    if (mode == 0) return;

    TQT(3);
    // 3. tau_max over free joints (kcm.py:325-326)
    const uint8_t *frozen = w.frozen + (size_t)b * D;
    double tmax = 0.0;
    if (mode == 1)
        for (int d = threadIdx.x; d < D; d += blockDim.x)
            if (!frozen[d]) tmax = fmax(tmax, fabs(tau[d]));

    // 4. energies: full-list halves summed in a fixed order
    const int n = c.n_atoms;
    const double *ea = w.e_atom + (size_t)b * n * 2;
    double se = 0.0, sv = 0.0, sc = 0.0, sp = 0.0, sp5 = 0.0;
    // (e_first: the cluster-pair kernel left its totals at atom 0 only)
    for (int a = threadIdx.x; a < n; a += blockDim.x) {
        if (f.solvation) sc += w.cav_atom[(size_t)b * n + a];
        if (e_first && a) continue;
        se += ea[2 * a]; sv += ea[2 * a + 1];
        const long long pc = w.pair_count[(size_t)b * n + a];
        sp += (double)(pc & 0xffffffffLL);
        sp5 += (double)(pc >> 32);
    }
    // one block reduction for all six (warp trees, then the warps in order: 2 barriers)
    {
        __shared__ double red6[32][6];
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
        double v[6] = {warp_max(tmax), warp_sum(se), warp_sum(sv), warp_sum(sc), warp_sum(sp), warp_sum(sp5)};
        __syncthreads();
        if (lane == 0)
            for (int q = 0; q < 6; ++q) red6[wid][q] = v[q];
        __syncthreads();
        for (int q = 0; q < 6; ++q) v[q] = red6[0][q];
        for (int w2 = 1; w2 < nw; ++w2) {
            v[0] = fmax(v[0], red6[w2][0]);
            for (int q = 1; q < 6; ++q) v[q] += red6[w2][q];
        }
        tmax = v[0]; se = v[1]; sv = v[2]; sc = v[3]; sp = v[4]; sp5 = v[5];
    }
    const double ge = 0.5 * se, gv = 0.5 * sv, gc = sc;
    if (mode == 2) {   // Field.evaluate: energies only
        if (threadIdx.x == 0) {
            double *e = w.energy + 3 * (size_t)b;
            e[0] = ge; e[1] = gv; e[2] = gc;
            if (st) { st->n_pairs = (long long)(0.5 * sp); st->n_pairs_vdw = (long long)(0.5 * sp5); }
        }
        return;
    }
    TQT(4);
    finish_iteration(c, w, step, b, tau, tmax, ge, gv, gc, sp, sp5, &stop_reason);
#ifdef TQ_TIMING
    TQT(5);
    if (b == 0 && threadIdx.x == 0)
        printf("TQT wrench %lld side %lld backbone %lld tmax+energies %lld step %lld total %lld\n", tk[1] - tk[0],
               tk[2] - tk[1], tk[3] - tk[2], tk[4] - tk[3], tk[5] - tk[4], tk[5] - tk[0]);
#endif
}

template <int NT>
__global__ void __launch_bounds__(NT, 1024 / NT)   // 64 registers: 4 CTAs of 256 per SM
torque_step_kernel(kf_chain_t c, kf_field_t f, TorqueArgs ta, kf_batch_t w, kf_step_t step, int mode,
                   int fuse_wrench, int e_first) {
    kf_pdl_wait();      // after the predecessor (programmatic launch: single trajectories)
    kf_pdl_trigger();
    extern __shared__ __align__(16) double wsm_dyn[];   // [L][6] when fuse_wrench
    torque_step_cta<NT>(c, f, ta, w, step, mode, fuse_wrench, e_first, blockIdx.x, wsm_dyn);
}

// ---- long chains: the same iteration over several CTAs per trajectory ------
//
// The backbone is cut into segments of TQ_SEG dofs (one CTA each).  Pass 1:
// each CTA runs the side chains attached in its segment and the segment-local
// blocked suffix scan; segment totals go to scratch.  Pass 2: each CTA adds the
// totals of the later segments, projects its backbone torques and reduces a
// partial tau_max and a slice of the energy sums.  Pass 3 (one CTA per
// trajectory) combines the partials in segment order and finishes the
// iteration.  scratch = fk_scratch ([B][n_seg][12]: segment total 6 |
// partials 6), free once forward kinematics has run.
#ifndef TQ_SEG_N
#define TQ_SEG_N 512
#endif
constexpr int TQ_SEG = TQ_SEG_N;   // <= the FK segment (they share fk_scratch rows)

__global__ void __launch_bounds__(TQ_THREADS)
torque_seg_kernel(kf_chain_t c, TorqueArgs ta, kf_batch_t w, int n_seg) {
    const int g = blockIdx.x, b = blockIdx.y;
    const kf_status_t *st = w.status + b;
    if (st->done || st->error) return;
    __shared__ double chunk[TQ_THREADS / 32][6];   // warp totals of the suffix scan
    __shared__ double red[32];
    const int L = c.n_links, D = c.n_dof, nb = c.n_bb;
    const double *T = ta.link_T + (size_t)b * L * KF_XF_STRIDE;
    const double *Wr = ta.wrench + (size_t)b * L * 6;
    double *suf = ta.bb_suffix + (size_t)b * nb * 6;
    double *tau = ta.tau + (size_t)b * D;
    const uint8_t *frozen = w.frozen + (size_t)b * D;
    const int k0 = g * TQ_SEG, k1 = min(nb, k0 + TQ_SEG);
    const int per = (k1 - k0 + blockDim.x - 1) / blockDim.x;
    const int lo = min(k1, k0 + (int)threadIdx.x * per), hi = min(k1, lo + per);
    W6 acc = w6_zero();
    double tmax = 0.0;
    for (int k = hi - 1; k >= lo; --k) {
        w6_add(acc, w6_load(Wr + 6 * c.bb_by_dof[k]));
        const int r = c.bb_side_res[k];
        if (r >= 0) {   // the residue's side chain: plain suffix in chi order (kcm.py:209-225)
            W6 agg = w6_zero();
            for (int e = c.chi_res_off[r + 1] - 1; e >= c.chi_res_off[r]; --e) {
                const int l = c.chi_links[e];
                w6_add(agg, w6_load(Wr + 6 * l));
                const int d = c.link_dof[l];
                const double t = project(T + KF_XF_STRIDE * l, agg);
                tau[d] = t;
                if (!frozen[d]) tmax = fmax(tmax, fabs(t));
            }
            w6_add(acc, agg);
        }
        w6_store(suf + 6 * k, acc);
    }
    W6 seg_total;
    const W6 later = w6_block_suffix(acc, chunk, seg_total);
    if (threadIdx.x + 1 < blockDim.x) {
        for (int k = lo; k < hi; ++k) {
            W6 s6 = w6_load(suf + 6 * k);
            w6_add(s6, later);
            w6_store(suf + 6 * k, s6);
        }
    }
    tmax = block_max(tmax, red);
    double *sc = w.fk_scratch + ((size_t)b * n_seg + g) * 12;
    if (threadIdx.x == 0) {
        w6_store(sc, seg_total);
        sc[6] = tmax;
    }
}

__global__ void __launch_bounds__(TQ_THREADS)
torque_seg_project_kernel(kf_chain_t c, kf_field_t f, TorqueArgs ta, kf_batch_t w, int n_seg, int e_first) {
    const int g = blockIdx.x, b = blockIdx.y;
    const kf_status_t *st = w.status + b;
    if (st->done || st->error) return;
    __shared__ double red[32];
    const int L = c.n_links, D = c.n_dof, nb = c.n_bb, n = c.n_atoms;
    const double *T = ta.link_T + (size_t)b * L * KF_XF_STRIDE;
    const double *suf = ta.bb_suffix + (size_t)b * nb * 6;
    double *tau = ta.tau + (size_t)b * D;
    const uint8_t *frozen = w.frozen + (size_t)b * D;
    double *sc = w.fk_scratch + (size_t)b * n_seg * 12;
    W6 later = w6_zero();
    for (int h = n_seg - 1; h > g; --h) w6_add(later, w6_load(sc + 12 * h));
    const int k0 = g * TQ_SEG, k1 = min(nb, k0 + TQ_SEG);
    double tmax = 0.0;
    for (int k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        const int l = c.bb_by_dof[k];
        W6 s6 = w6_load(suf + 6 * k);
        w6_add(s6, later);
        const int d = c.link_dof[l];
        const double t = project(T + KF_XF_STRIDE * l, s6);
        tau[d] = t;
        if (!frozen[d]) tmax = fmax(tmax, fabs(t));
    }
    tmax = block_max(tmax, red);
    // this CTA's slice of the energy sums
    const int a0 = (int)((long long)n * g / n_seg), a1 = (int)((long long)n * (g + 1) / n_seg);
    const double *ea = w.e_atom + (size_t)b * n * 2;
    double se = 0.0, sv = 0.0, scv = 0.0, sp = 0.0, sp5 = 0.0;
    for (int a = a0 + threadIdx.x; a < a1; a += blockDim.x) {
        if (f.solvation) scv += w.cav_atom[(size_t)b * n + a];
        if (e_first && a) continue;
        se += ea[2 * a]; sv += ea[2 * a + 1];
        const long long pc = w.pair_count[(size_t)b * n + a];
        sp += (double)(pc & 0xffffffffLL);
        sp5 += (double)(pc >> 32);
    }
    se = block_sum(se, red);
    sv = block_sum(sv, red);
    scv = block_sum(scv, red);
    sp = block_sum(sp, red);
    sp5 = block_sum(sp5, red);
    if (threadIdx.x == 0) {
        double *p = sc + 12 * g + 6;
        p[0] = fmax(p[0], tmax);   // p[0]: side-chain max from pass 1
        p[1] = se; p[2] = sv; p[3] = scv; p[4] = sp; p[5] = sp5;
    }
}

__global__ void __launch_bounds__(TQ_THREADS)
torque_seg_finish_kernel(kf_chain_t c, TorqueArgs ta, kf_batch_t w, kf_step_t step, int n_seg) {
    const int b = blockIdx.x;
    kf_status_t *st = w.status + b;
    double *sc = w.fk_scratch + (size_t)b * n_seg * 12;
    // decision for the step pass in sc[0][0..2]: (reason, tau_max, iteration); -1 = no record, no step
    if (st->done || st->error) {
        if (threadIdx.x == 0) {
            if (!st->done) st->done = 1;   // domain error this iteration: freeze
            sc[0] = -1.0;
        }
        return;
    }
    if (threadIdx.x != 0) return;
    double tmax = 0.0, se = 0.0, sv = 0.0, scv = 0.0, sp = 0.0, sp5 = 0.0;
    for (int g = 0; g < n_seg; ++g) {   // fixed order: deterministic
        const double *p = sc + 12 * g + 6;
        tmax = fmax(tmax, p[0]);
        se += p[1]; sv += p[2]; scv += p[3]; sp += p[4]; sp5 += p[5];
    }
    const int it = st->iter;
    const int reason = decide_iteration(w, step, b, it, tmax, 0.5 * se, 0.5 * sv, scv, sp, sp5);
    sc[0] = (double)reason; sc[1] = tmax; sc[2] = (double)it;
    close_iteration(st, step, it, reason);
}

// Theta records and the compliance step, dof ranges spread over n_seg CTAs.
__global__ void __launch_bounds__(TQ_THREADS)
torque_seg_step_kernel(kf_chain_t c, TorqueArgs ta, kf_batch_t w, kf_step_t step, int n_seg) {
    const int g = blockIdx.x, b = blockIdx.y;
    const double *sc = w.fk_scratch + (size_t)b * n_seg * 12;
    const double code = sc[0];
    if (code < 0.0) return;
    const int D = c.n_dof;
    const int d0 = (int)((long long)D * g / n_seg), d1 = (int)((long long)D * (g + 1) / n_seg);
    step_dofs(w, step, b, D, (int)sc[2], (int)code, ta.tau + (size_t)b * D, sc[1], d0, d1, threadIdx.x,
              blockDim.x);
}

// kcm_step for the API (B = 1): deltas and theta' (kcm.py:264-274).
__global__ void kcm_step_api_kernel(const double *tau, const double *theta, const uint8_t *frozen, int D,
                                    double kappa, double *theta_out, double *deltas) {
    __shared__ double red[32];
    double tmax = 0.0;
    for (int d = threadIdx.x; d < D; d += blockDim.x)
        if (!frozen[d]) tmax = fmax(tmax, fabs(tau[d]));
    tmax = block_max(tmax, red);
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
        double delta = 0.0;
        if (tmax != 0.0 && !frozen[d]) delta = __ddiv_rn(xmul(kappa, tau[d]), tmax);
        deltas[d] = delta;
        theta_out[d] = tmax == 0.0 ? theta[d] : np_mod360(np_mod360(xadd(theta[d], delta)));
    }
}

}  // namespace

int kf_cluster_path(const kf_field_t *f, const kf_batch_t *w, int n);

int kf_wrench_launch(const kf_chain_t *c, int B, const double *pos, const double *forces, double *wrench,
                     const kf_status_t *status, cudaStream_t s) {
    const long long total = (long long)B * c->n_links;
    wrench_kernel<<<kf_blocks(total, 128), 128, 0, s>>>(*c, B, pos, forces, wrench, status);
    KF_LAUNCH_CHECK("wrench_kernel");
    return 0;
}

int kf_torque_launch(const kf_chain_t *c, const kf_field_t *f, kf_batch_t *w, const double *link_T,
                     const double *wrench, double *side_tot, double *bb_suffix, double *tau,
                     const kf_step_t *step, int mode, cudaStream_t s, int fuse_wrench) {
    TorqueArgs ta{link_T, wrench, side_tot, bb_suffix, tau};
    kf_step_t st{};
    if (step) st = *step;
    kf_field_t fz{};
    if (f) fz = *f;
    const int n_seg = (c->n_bb + TQ_SEG - 1) / TQ_SEG;
    const int e_first = (f && mode != 0) ? kf_cluster_path(f, w, c->n_atoms) : 0;
    if (mode == 1 && n_seg > 1 && w->B * n_seg <= 4 * 148 && w->fk_scratch && bb_suffix) {
        if (fuse_wrench &&
            kf_wrench_launch(c, w->B, w->pos, w->forces, const_cast<double *>(wrench), w->status, s)) return 1;
        torque_seg_kernel<<<dim3(n_seg, w->B), TQ_THREADS, 0, s>>>(*c, ta, *w, n_seg);
        KF_LAUNCH_CHECK("torque_seg_kernel");
        torque_seg_project_kernel<<<dim3(n_seg, w->B), TQ_THREADS, 0, s>>>(*c, fz, ta, *w, n_seg, e_first);
        KF_LAUNCH_CHECK("torque_seg_project_kernel");
        torque_seg_finish_kernel<<<w->B, 32, 0, s>>>(*c, ta, *w, st, n_seg);
        KF_LAUNCH_CHECK("torque_seg_finish_kernel");
        torque_seg_step_kernel<<<dim3(n_seg, w->B), TQ_THREADS, 0, s>>>(*c, ta, *w, st, n_seg);
        KF_LAUNCH_CHECK("torque_seg_step_kernel");
        return 0;
    }
    // a fold iteration computes its own wrenches (pos, forces of this batch) in
    // shared memory when they fit; otherwise the separate wrench pass
    const size_t wsm = (size_t)c->n_links * 6 * sizeof(double);
    const bool fuse = fuse_wrench && wsm <= 96 * 1024;
    if (fuse_wrench && !fuse) {
        if (kf_wrench_launch(c, w->B, w->pos, w->forces, const_cast<double *>(wrench), w->status, s)) return 1;
    }
    // one CTA per trajectory: 512 threads for small batches (the chain's latency is the
    // iteration's), 256 from 64 trajectories: with the fold loop's graph branches a
    // torque CTA shares the GPU with other branches' pair CTAs, and its registers x
    // time are what it takes from them (C5 step: 256 0.629 vs 512 0.655 ms; B = 128 as
    // 2 x 64: 0.128 vs 0.130; 128 threads 0.624 at C5 but 0.148 at B = 128)
#ifndef TQ_NARROW
#define TQ_NARROW (TQ_THREADS / 2)
#endif
#ifndef TQ_WIDE_B
#define TQ_WIDE_B 64
#endif
    const bool wide = w->B < TQ_WIDE_B;
    auto kern = wide ? torque_step_kernel<TQ_THREADS> : torque_step_kernel<TQ_NARROW>;
    if (fuse) {
        static size_t opted[2] = {0, 0};
        if (wsm > opted[wide]) {
            KF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm), "torque smem");
            opted[wide] = wsm;
        }
    }
    (void)kf_launch(w->B < KF_PDL_B, kern, dim3(w->B), dim3(wide ? TQ_THREADS : TQ_NARROW), fuse ? wsm : 0, s, *c, fz, ta,
                    *w, st, mode, fuse ? 1 : 0, e_first);
    KF_LAUNCH_CHECK("torque_step_kernel");
    return 0;
}

int kf_kcm_step_launch(const double *tau, const double *theta, const uint8_t *frozen, int D, double kappa,
                       double *theta_out, double *deltas, cudaStream_t s) {
    kcm_step_api_kernel<<<1, 512, 0, s>>>(tau, theta, frozen, D, kappa, theta_out, deltas);
    KF_LAUNCH_CHECK("kcm_step_api_kernel");
    return 0;
}
