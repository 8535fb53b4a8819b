// Forward kinematics as a parallel scan of rigid transforms (K4).
//
// Reference: chain.kinematic_state (/root/reference/pkg/src/kinefold/chain.py:
// 240-261) walks links sequentially: M_l = M_parent R(axis0_l, theta_l),
// P_l = P_parent + M_parent body0_parent, pos_a = P_l + M_l (zp_a - point0_l).
// Written as affine maps that is T_l = T_parent o A_l with
// A_l = (R(axis0_l, theta_l), body0_parent), an associative composition, so the
// backbone path (phi/psi links) is a prefix scan and the <= 4-deep side
// branches follow level by level.  fp64 throughout; the scan re-associates the
// products, so positions differ from the sequential walk at the 1e-13 A level.
#include "kf_common.cuh"
#ifdef FK_TIMING
#include <cstdio>
#endif

namespace {

constexpr int FK_THREADS = 256;

// Rodrigues R = I + sin(t) K + (1 - cos(t)) K^2 (geometry.py:26-41), t in radians
// from degrees as math.radians does (x * (pi / 180)).
KF_DEV Xf local_transform_v(double x, double y, double z, double theta_deg, double bx, double by, double bz) {
    const double deg2rad = 0.017453292519943295;
    double s, c;
    sincos(theta_deg * deg2rad, &s, &c);
    const double omc = 1.0 - c;
    Xf t;
    // K^2 = a a^T - |a|^2 I, written out as the reference's (k @ k) entries
    const double k00 = -(y * y + z * z), k11 = -(x * x + z * z), k22 = -(x * x + y * y);
    const double k01 = x * y, k02 = x * z, k12 = y * z;
    t.m[0] = 1.0 + omc * k00;   t.m[1] = -s * z + omc * k01; t.m[2] = s * y + omc * k02;
    t.m[3] = s * z + omc * k01; t.m[4] = 1.0 + omc * k11;    t.m[5] = -s * x + omc * k12;
    t.m[6] = -s * y + omc * k02; t.m[7] = s * x + omc * k12; t.m[8] = 1.0 + omc * k22;
    t.p[0] = bx; t.p[1] = by; t.p[2] = bz;
    return t;
}
KF_DEV Xf local_transform(const double *axis, double theta_deg, const double *body_parent) {
    return local_transform_v(axis[0], axis[1], axis[2], theta_deg, body_parent[0], body_parent[1], body_parent[2]);
}

// Block-wide scan of the threads' transforms in thread order (composition is
// associative, not commutative): warp-level Hillis-Steele on registers by
// shuffles, then the warp totals (wtot, one row per warp) composed in warp
// order.  Returns the thread's exclusive prefix (identity for thread 0) and,
// in incl, its inclusive one.  Two block barriers instead of two per step.
KF_DEV Xf xf_block_scan(const Xf &acc, double (*wtot)[12], Xf &incl) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    incl = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        Xf up;
#pragma unroll
        for (int q = 0; q < 9; ++q) up.m[q] = __shfl_up_sync(0xffffffffu, incl.m[q], o);
#pragma unroll
        for (int q = 0; q < 3; ++q) up.p[q] = __shfl_up_sync(0xffffffffu, incl.p[q], o);
        if (lane >= o) incl = xf_compose(up, incl);
    }
    __syncthreads();
    if (lane == 31) xf_store(wtot[wid], incl);
    __syncthreads();
    Xf wpre = xf_identity();
    for (int w2 = 0; w2 < wid; ++w2) wpre = xf_compose(wpre, xf_load(wtot[w2]));
    Xf pre;
#pragma unroll
    for (int q = 0; q < 9; ++q) pre.m[q] = __shfl_up_sync(0xffffffffu, incl.m[q], 1);
#pragma unroll
    for (int q = 0; q < 3; ++q) pre.p[q] = __shfl_up_sync(0xffffffffu, incl.p[q], 1);
    if (wid > 0) incl = xf_compose(wpre, incl);
    if (lane == 0) pre = wpre;
    else if (wid > 0) pre = xf_compose(wpre, pre);
    return pre;
}

// One CTA per trajectory: local transforms, blocked backbone scan, side levels.
__global__ void __launch_bounds__(FK_THREADS)
fk_scan_kernel(kf_chain_t c, const double *__restrict__ theta_all, double *__restrict__ T_all,
               const kf_status_t *__restrict__ status) {
    const int b = blockIdx.x;
    if (status && status[b].done) return;
    const int L = c.n_links, D = c.n_dof;
    const double *theta = theta_all + (size_t)b * D;
    double *T = T_all + (size_t)b * L * KF_XF_STRIDE;
    __shared__ double chunk[FK_THREADS / 32][12];   // warp totals of the block scan

    // 1. local transforms (ground = identity)
    for (int l = threadIdx.x; l < L; l += blockDim.x) {
        Xf a;
        if (l == 0 || c.link_dof[l] < 0) {
            a = xf_identity();
        } else {
            const int p = c.link_parent[l];
            a = local_transform(c.link_axis0 + 3 * l, theta[c.link_dof[l]], c.link_body0 + 3 * p);
        }
        xf_store(T + KF_XF_STRIDE * l, a);
    }
    __syncthreads();

    // 2. backbone path: per-thread chunk prefix, then a scan of chunk totals
    const int nb = c.n_bb;
    const int per = (nb + blockDim.x - 1) / blockDim.x;
    const int lo = min(nb, (int)threadIdx.x * per), hi = min(nb, lo + per);
    Xf acc = xf_identity();
    for (int k = lo; k < hi; ++k) {
        double *slot = T + KF_XF_STRIDE * c.bb_order[k];
        acc = xf_compose(acc, xf_load(slot));
        xf_store(slot, acc);
    }
    Xf incl;
    const Xf pre = xf_block_scan(acc, chunk, incl);
    if (threadIdx.x > 0 && lo < hi) {
        for (int k = lo; k < hi; ++k) {
            double *slot = T + KF_XF_STRIDE * c.bb_order[k];
            xf_store(slot, xf_compose(pre, xf_load(slot)));
        }
    }
    __syncthreads();

    // 3. side branches, one depth level at a time
    for (int d = 0; d < c.side_depth; ++d) {
        for (int k = c.side_depth_off[d] + threadIdx.x; k < c.side_depth_off[d + 1]; k += blockDim.x) {
            const int l = c.side_order[k];
            double *slot = T + KF_XF_STRIDE * l;
            xf_store(slot, xf_compose(xf_load(T + KF_XF_STRIDE * c.link_parent[l]), xf_load(slot)));
        }
        __syncthreads();
    }

    // 4. current joint axes U_l = M_l axis0_l (chain.py:257); ground keeps 0
    for (int l = threadIdx.x; l < L; l += blockDim.x) {
        double *slot = T + KF_XF_STRIDE * l;
        const double *a = c.link_axis0 + 3 * l;
        for (int r = 0; r < 3; ++r)
            slot[12 + r] = (l == 0 || c.link_dof[l] < 0)
                               ? 0.0 : slot[3 * r] * a[0] + slot[3 * r + 1] * a[1] + slot[3 * r + 2] * a[2];
        slot[15] = 0.0;
    }
}

// ---- short chains: the whole iteration's FK in shared memory ----------------
// Same operations and association as fk_scan_kernel, but the link transforms
// live in shared memory (12 doubles each) until the final write of T (with
// the joint axes) and of the atom positions, which this kernel also computes:
// one global write per link and per atom instead of several read-modify-writes.
#ifndef FKS_THREADS_N
#define FKS_THREADS_N 128
#endif
constexpr int FKS_THREADS = FKS_THREADS_N;
constexpr int FKS_STRIDE = 12;

// The whole FK of trajectory b by one CTA of NT threads in S ([L][12] doubles, then
// the walk tables): also the first phase of the fused fold iteration (kf_cluster.cu).
// full_t = 0 (the fold loop): only the second half of each T row is written, which
// holds the joint point and axis the torque kernel projects with (rows 8-15:
// M[8], P, U, pad); the API's kinematic_state asks for the whole row.
#ifdef FK_TIMING   // phase clocks of CTA 0 (measurement builds only)
#define FKT(k) do { if (b == 0 && threadIdx.x == 0) tk[k] = clock64(); } while (0)
#else
#define FKT(k) do { } while (0)
#endif
template <int NT>
KF_DEV void fk_smem_cta(const kf_chain_t &c, int b, const double *__restrict__ theta_all,
                        double *__restrict__ T_all, double *__restrict__ pos_all, double *__restrict__ S,
                        int full_t = 1) {
    __shared__ double chunk[NT / 32][12];   // warp totals of the block scan
    __shared__ int sh_doff[8];               // side-level offsets (side_depth <= 7 staged)
#ifdef FK_TIMING
    long long tk[8];
#endif
    FKT(0);
    const int L = c.n_links, D = c.n_dof, n = c.n_atoms, nb = c.n_bb, ns = c.n_side;
    const double *theta = theta_all + (size_t)b * D;
    // the chain tables the serial phases walk, staged once (one global round trip
    // instead of one per dependent step): parent, dof, backbone order, side order
    int *sh_par = reinterpret_cast<int *>(S + FKS_STRIDE * L), *sh_dof = sh_par + L, *sh_bb = sh_dof + L,
        *sh_side = sh_bb + nb;
    for (int k = threadIdx.x; k < nb; k += blockDim.x) sh_bb[k] = c.bb_order[k];
    for (int k = threadIdx.x; k < ns; k += blockDim.x) sh_side[k] = c.side_order[k];
    const int nd = min(c.side_depth, 7);
    if ((int)threadIdx.x <= nd) sh_doff[threadIdx.x] = c.side_depth_off[threadIdx.x];

    {
        // local transforms; the chain tables, axes, parent offsets and angles of U
        // links per thread are loaded ahead of the math (two dependent rounds, not 2 U)
        const int32_t *__restrict__ link_dof = c.link_dof;
        const int32_t *__restrict__ link_parent = c.link_parent;
        const double *__restrict__ axis0 = c.link_axis0;
        const double *__restrict__ body0 = c.link_body0;
        constexpr int U = 4;
        for (int l0 = threadIdx.x; l0 < L; l0 += U * blockDim.x) {
            int dof[U], par[U];
            double th[U], ax[U][3], bo[U][3];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int l = l0 + u * blockDim.x;
                dof[u] = (l < L && l != 0) ? link_dof[l] : -1;
                par[u] = (l < L && l != 0) ? link_parent[l] : 0;
#pragma unroll
                for (int q = 0; q < 3; ++q) ax[u][q] = l < L ? axis0[3 * l + q] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                th[u] = dof[u] >= 0 ? theta[dof[u]] : 0.0;
#pragma unroll
                for (int q = 0; q < 3; ++q) bo[u][q] = dof[u] >= 0 ? body0[3 * par[u] + q] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int l = l0 + u * blockDim.x;
                if (l >= L) break;
                sh_dof[l] = dof[u];
                sh_par[l] = par[u];
                const Xf a = dof[u] < 0 ? xf_identity()
                                        : local_transform_v(ax[u][0], ax[u][1], ax[u][2], th[u], bo[u][0], bo[u][1],
                                                            bo[u][2]);
                xf_store(S + FKS_STRIDE * l, a);
            }
        }
    }
    __syncthreads();
    FKT(1);

    const int per = (nb + blockDim.x - 1) / blockDim.x;
    const int lo = min(nb, (int)threadIdx.x * per), hi = min(nb, lo + per);
    Xf acc = xf_identity();
    for (int k = lo; k < hi; ++k) {
        double *slot = S + FKS_STRIDE * sh_bb[k];
        acc = xf_compose(acc, xf_load(slot));
        xf_store(slot, acc);
    }
    Xf incl;
    const Xf pre = xf_block_scan(acc, chunk, incl);
    if (threadIdx.x > 0 && lo < hi) {
        for (int k = lo; k < hi; ++k) {
            double *slot = S + FKS_STRIDE * sh_bb[k];
            xf_store(slot, xf_compose(pre, xf_load(slot)));
        }
    }
    __syncthreads();
    FKT(2);
    for (int d = 0; d < c.side_depth; ++d) {
        const int k0 = d < nd ? sh_doff[d] : c.side_depth_off[d];
        const int k1 = d + 1 <= nd ? sh_doff[d + 1] : c.side_depth_off[d + 1];
        for (int k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
            const int l = sh_side[k];
            double *slot = S + FKS_STRIDE * l;
            xf_store(slot, xf_compose(xf_load(S + FKS_STRIDE * sh_par[l]), xf_load(slot)));
        }
        __syncthreads();
    }
    FKT(3);
    // T with the current joint axes U_l = M_l axis0_l (chain.py:257); ground keeps 0.
    // The axis loads of TU links per thread are issued ahead of the stores.
    double *__restrict__ T = T_all + (size_t)b * L * KF_XF_STRIDE;
    const double *__restrict__ axis0 = c.link_axis0;
    constexpr int TU = 4;
    for (int l0 = threadIdx.x; l0 < L; l0 += TU * blockDim.x) {
        double ax[TU][3];
#pragma unroll
        for (int u = 0; u < TU; ++u) {
            const int l = l0 + u * blockDim.x;
#pragma unroll
            for (int q = 0; q < 3; ++q) ax[u][q] = l < L ? axis0[3 * l + q] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < TU; ++u) {
            const int l = l0 + u * blockDim.x;
            if (l >= L) break;
            const double *src = S + FKS_STRIDE * l;
            double2 *d2 = reinterpret_cast<double2 *>(T + (size_t)KF_XF_STRIDE * l);
            const bool joint = l != 0 && sh_dof[l] >= 0;
            double v[KF_XF_STRIDE];
#pragma unroll
            for (int q = 0; q < 12; ++q) v[q] = src[q];
#pragma unroll
            for (int r = 0; r < 3; ++r)
                v[12 + r] = joint ? v[3 * r] * ax[u][0] + v[3 * r + 1] * ax[u][1] + v[3 * r + 2] * ax[u][2] : 0.0;
            v[15] = 0.0;
#pragma unroll
            for (int q = 0; q < KF_XF_STRIDE / 2; ++q)
                if (full_t || q >= 4) d2[q] = make_double2(v[2 * q], v[2 * q + 1]);
        }
    }
#ifdef FK_TIMING
    __syncthreads();
#endif
    FKT(4);
    // positions pos_a = P_l + M_l zrel_a (fk_positions_kernel's arithmetic);
    // the chain tables are loaded ahead of the stores (no aliasing with pos)
    double *__restrict__ pos = pos_all + (size_t)b * n * 3;
    const int32_t *__restrict__ atom_link = c.atom_link;
    const double *__restrict__ zrel = c.atom_zrel;
    constexpr int U = 4;
    for (int a0 = threadIdx.x; a0 < n; a0 += U * blockDim.x) {
        int lk[U];
        double z[U][3];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int a = a0 + u * blockDim.x;
            lk[u] = a < n ? atom_link[a] : 0;
            for (int q = 0; q < 3; ++q) z[u][q] = a < n ? zrel[3 * a + q] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int a = a0 + u * blockDim.x;
            if (a >= n) break;
            const double *t = S + FKS_STRIDE * lk[u];
            pos[3 * a] = t[9] + (t[0] * z[u][0] + t[1] * z[u][1] + t[2] * z[u][2]);
            pos[3 * a + 1] = t[10] + (t[3] * z[u][0] + t[4] * z[u][1] + t[5] * z[u][2]);
            pos[3 * a + 2] = t[11] + (t[6] * z[u][0] + t[7] * z[u][1] + t[8] * z[u][2]);
        }
    }
#ifdef FK_TIMING
    __syncthreads();
    FKT(5);
    if (b == 0 && threadIdx.x == 0)
        printf("FKT tables+local %lld bbscan %lld side %lld Twrite %lld positions %lld total %lld\n", tk[1] - tk[0],
               tk[2] - tk[1], tk[3] - tk[2], tk[4] - tk[3], tk[5] - tk[4], tk[5] - tk[0]);
#endif
}

__global__ void __launch_bounds__(FKS_THREADS)
fk_smem_kernel(const __grid_constant__ kf_chain_t c, const double *__restrict__ theta_all,
               double *__restrict__ T_all, double *__restrict__ pos_all, const kf_status_t *__restrict__ status,
               int full_t) {
    kf_pdl_wait();      // after the predecessor (programmatic launch: single trajectories)
    kf_pdl_trigger();
    const int b = blockIdx.x;
    if (status && status[b].done) return;
    extern __shared__ __align__(16) double S[];     // [L][12], then the int tables
    fk_smem_cta<FKS_THREADS>(c, b, theta_all, T_all, pos_all, S, full_t);
}

inline size_t fk_smem_bytes(const kf_chain_t &c) {
    return (size_t)c.n_links * FKS_STRIDE * sizeof(double) +
           sizeof(int32_t) * (2 * (size_t)c.n_links + c.n_bb + c.n_side);
}

// ---- long chains: the backbone scan spread over many CTAs --------------------
// Three phases per trajectory: (1) every CTA scans a SEG-link segment of the
// backbone in place (local transforms computed on the fly) and publishes the
// segment total; (2) one CTA scans the segment totals; (3) every CTA applies
// its exclusive prefix and computes the segment's axes.  Side links then
// compose their <= 4 ancestors from the (final) backbone transform directly.
#ifndef FK_SEG
#define FK_SEG 512
#endif
constexpr int SEG = FK_SEG;                 // kf_common: KF_BB_SEG (scratch rows)
constexpr int SEG_PER = SEG / FK_THREADS;   // links per thread

__global__ void __launch_bounds__(FK_THREADS)
fk_seg_scan_kernel(kf_chain_t c, const double *__restrict__ theta_all, double *__restrict__ T_all,
                   double *__restrict__ seg_tot, int n_seg, const kf_status_t *__restrict__ status) {
    const int b = blockIdx.y, g = blockIdx.x;
    if (status && status[b].done) return;
    const int L = c.n_links, D = c.n_dof, nb = c.n_bb;
    const double *theta = theta_all + (size_t)b * D;
    double *T = T_all + (size_t)b * L * KF_XF_STRIDE;
    __shared__ double chunk[FK_THREADS / 32][12];   // warp totals of the block scan
    const int lo = min(nb, g * SEG + (int)threadIdx.x * SEG_PER), hi = min(nb, lo + SEG_PER);
    Xf acc = xf_identity();
    for (int k = lo; k < hi; ++k) {
        const int l = c.bb_order[k];
        const Xf loc = local_transform(c.link_axis0 + 3 * l, theta[c.link_dof[l]],
                                       c.link_body0 + 3 * c.link_parent[l]);
        acc = xf_compose(acc, loc);
        xf_store(T + KF_XF_STRIDE * l, acc);
    }
    Xf incl;
    const Xf pre = xf_block_scan(acc, chunk, incl);
    if (threadIdx.x > 0 && lo < hi) {
        for (int k = lo; k < hi; ++k) {
            double *slot = T + KF_XF_STRIDE * c.bb_order[k];
            xf_store(slot, xf_compose(pre, xf_load(slot)));
        }
    }
    if (threadIdx.x == blockDim.x - 1) xf_store(seg_tot + ((size_t)b * n_seg + g) * 12, incl);
}

// exclusive prefix of the segment totals, in place (one thread per trajectory: few segments)
// Exclusive prefix of the segment totals, one CTA per trajectory (thread =
// segment): Hillis-Steele over the compositions in shared memory.
__global__ void fk_seg_prefix_kernel(double *__restrict__ seg_tot, int n_seg, int B,
                                     const kf_status_t *__restrict__ status) {
    const int b = blockIdx.x, g = threadIdx.x;
    if (status && status[b].done) return;
    extern __shared__ double pre[];   // [blockDim][12]
    double *slot = seg_tot + ((size_t)b * n_seg + g) * 12;
    const Xf mine = g < n_seg ? xf_load(slot) : xf_identity();
    xf_store(pre + 12 * g, mine);
    __syncthreads();
    for (int off = 1; off < (int)blockDim.x; off <<= 1) {
        Xf r = xf_load(pre + 12 * g);
        if (g >= off) r = xf_compose(xf_load(pre + 12 * (g - off)), r);
        __syncthreads();
        xf_store(pre + 12 * g, r);
        __syncthreads();
    }
    if (g < n_seg) xf_store(slot, g > 0 ? xf_load(pre + 12 * (g - 1)) : xf_identity());
}

KF_DEV void store_axis(double *slot, const double *axis0) {
    for (int r = 0; r < 3; ++r)
        slot[12 + r] = slot[3 * r] * axis0[0] + slot[3 * r + 1] * axis0[1] + slot[3 * r + 2] * axis0[2];
    slot[15] = 0.0;
}

__global__ void fk_seg_apply_kernel(kf_chain_t c, double *__restrict__ T_all, const double *__restrict__ seg_tot,
                                    int n_seg, int B, const kf_status_t *__restrict__ status) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int nb = c.n_bb;
    if (gid >= (long long)B * nb) return;
    const int b = (int)(gid / nb), k = (int)(gid % nb);
    if (status && status[b].done) return;
    double *T = T_all + (size_t)b * c.n_links * KF_XF_STRIDE;
    const int l = c.bb_order[k];
    double *slot = T + KF_XF_STRIDE * l;
    const int g = k / SEG;
    if (g > 0) xf_store(slot, xf_compose(xf_load(seg_tot + ((size_t)b * n_seg + g) * 12), xf_load(slot)));
    store_axis(slot, c.link_axis0 + 3 * l);
}

// side links: compose the chain of (<= 4) side ancestors onto the backbone link
__global__ void fk_side_kernel(kf_chain_t c, const double *__restrict__ theta_all, double *__restrict__ T_all,
                               int B, const kf_status_t *__restrict__ status) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int ns = c.n_side;
    if (gid >= (long long)B * (ns + 1)) return;
    const int b = (int)(gid / (ns + 1)), k = (int)(gid % (ns + 1));
    if (status && status[b].done) return;
    double *T = T_all + (size_t)b * c.n_links * KF_XF_STRIDE;
    if (k == ns) {   // ground
        Xf id = xf_identity();
        xf_store(T, id);
        for (int r = 0; r < 4; ++r) T[12 + r] = 0.0;
        return;
    }
    const double *theta = theta_all + (size_t)b * c.n_dof;
    const int l = c.side_order[k];
    int chain_l[8];
    int depth = 0, cur = l;
    while (cur > 0 && depth < 8) {   // climb to the first backbone (or ground) ancestor
        // backbone links carry dofs 0..n_bb-1 (validated on the host), side links the rest
        const bool is_side = c.link_dof[cur] >= c.n_bb;
        if (!is_side) break;
        chain_l[depth++] = cur;
        cur = c.link_parent[cur];
    }
    Xf acc = cur > 0 ? xf_load(T + KF_XF_STRIDE * cur) : xf_identity();
    for (int d = depth - 1; d >= 0; --d) {
        const int q = chain_l[d];
        acc = xf_compose(acc, local_transform(c.link_axis0 + 3 * q, theta[c.link_dof[q]],
                                              c.link_body0 + 3 * c.link_parent[q]));
    }
    double *slot = T + KF_XF_STRIDE * l;
    xf_store(slot, acc);
    store_axis(slot, c.link_axis0 + 3 * l);
}

// pos_a = P_l + M_l zrel_a over every (trajectory, atom)
__global__ void fk_positions_kernel(kf_chain_t c, int B, const double *__restrict__ T_all,
                                    double *__restrict__ pos_all,
                                    const kf_status_t *__restrict__ status) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int n = c.n_atoms;
    if (gid >= (long long)B * n) return;
    const int b = (int)(gid / n), a = (int)(gid % n);
    if (status && status[b].done) return;
    const double *t = T_all + ((size_t)b * c.n_links + c.atom_link[a]) * KF_XF_STRIDE;
    const double zx = c.atom_zrel[3 * a], zy = c.atom_zrel[3 * a + 1], zz = c.atom_zrel[3 * a + 2];
    double *out = pos_all + 3 * gid;
    out[0] = t[9] + (t[0] * zx + t[1] * zy + t[2] * zz);
    out[1] = t[10] + (t[3] * zx + t[4] * zy + t[5] * zz);
    out[2] = t[11] + (t[6] * zx + t[7] * zy + t[8] * zz);
}

}  // namespace

int kf_fk_launch(const kf_chain_t *c, kf_batch_t *w, const kf_status_t *status, cudaStream_t s, int full_t) {
    const int n_seg = (c->n_bb + SEG - 1) / SEG;
    const size_t smem = (size_t)c->n_links * FKS_STRIDE * sizeof(double) +
                        sizeof(int32_t) * (2 * (size_t)c->n_links + c->n_bb + c->n_side);
    if (smem <= 110 * 1024) {   // whole chain (transforms + walk tables) in one CTA's shared memory
        static size_t opted = 0;
        if (smem > opted) {
            KF_CUDA(cudaFuncSetAttribute(fk_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                    "fk smem");
            opted = smem;
        }
        (void)kf_launch(w->B < KF_PDL_B, fk_smem_kernel, dim3(w->B), dim3(FKS_THREADS), smem, s, *c,
                        (const double *)w->theta, w->link_T, w->pos, status, full_t);
        KF_LAUNCH_CHECK("fk_smem_kernel");
        return 0;
    }
    if (n_seg > 1 && w->B * n_seg <= 4 * 148 && w->fk_scratch) {
        // long chain, few trajectories: multi-CTA backbone scan
        fk_seg_scan_kernel<<<dim3(n_seg, w->B), FK_THREADS, 0, s>>>(*c, w->theta, w->link_T, w->fk_scratch, n_seg,
                                                                     status);
        KF_LAUNCH_CHECK("fk_seg_scan_kernel");
        const int pt = (n_seg + 31) / 32 * 32;
        fk_seg_prefix_kernel<<<w->B, pt, (size_t)pt * 12 * sizeof(double), s>>>(w->fk_scratch, n_seg, w->B, status);
        KF_LAUNCH_CHECK("fk_seg_prefix_kernel");
        fk_seg_apply_kernel<<<kf_blocks((long long)w->B * c->n_bb, 256), 256, 0, s>>>(*c, w->link_T, w->fk_scratch,
                                                                                     n_seg, w->B, status);
        KF_LAUNCH_CHECK("fk_seg_apply_kernel");
        fk_side_kernel<<<kf_blocks((long long)w->B * (c->n_side + 1), 256), 256, 0, s>>>(*c, w->theta, w->link_T,
                                                                                         w->B, status);
        KF_LAUNCH_CHECK("fk_side_kernel");
    } else {
        fk_scan_kernel<<<w->B, FK_THREADS, 0, s>>>(*c, w->theta, w->link_T, status);
        KF_LAUNCH_CHECK("fk_scan_kernel");
    }
    const long long total = (long long)w->B * c->n_atoms;
    if (total > 0) {
        fk_positions_kernel<<<kf_blocks(total, 256), 256, 0, s>>>(*c, w->B, w->link_T, w->pos, status);
        KF_LAUNCH_CHECK("fk_positions_kernel");
    }
    return 0;
}
