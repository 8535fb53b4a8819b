// Cavity solvation by sample enumeration (K5): Algorithm 1 of the paper,
// steps 1 (exposure states) and 2 (forward-difference forces), fused.
//
// Reference: solvation.sasa_pass (/root/reference/pkg/src/kinefold/
// solvation.py:135-181) and solvation_forces (:194-255).  Every coverage test
// repeats the reference's fp64 operations in its order — sample point
// r_i + (R_off_i * q_k), diff = p - r_j (or p - (r_j + dr) for the displaced
// neighbour), d2 = (dx*dx + dy*dy) + dz*dz, compared with R_off_j^2 — and the
// forces accumulate in the reference's int64 fixed point, so states, exposure
// counts and forces are bit-identical and independent of thread schedule.
//
// One CTA per atom i: the reachable neighbours (|r_i - r_j| <= R_off_i +
// R_off_j + dr + slack; no farther atom can cover or, displaced by dr, newly
// cover a sample) are staged in shared memory; one thread per sample counts
// cover up to the clamp at 2 (the state is independent of neighbour order,
// so the scan stops at the second cover) and immediately runs step 2 for
// that sample; neighbour-side events go to per-slot shared int64 counters
// flushed once to global memory, the atom's own to a block reduction.
#include <cstdlib>

#include "kf_common.cuh"

#ifdef SOLV_STATS
__device__ unsigned long long g_solv_stats[8];
#define SSTAT(k, v) atomicAdd(&g_solv_stats[k], (unsigned long long)(v))
#else
#define SSTAT(k, v)
#endif

namespace {

constexpr int SOLV_THREADS = 256;
constexpr int SOLV_MAX_GROUPS = 128;   // sample groups tracked in shared memory (N <= 4096)
#ifndef SOLV_GROUP_THREADS
#define SOLV_GROUP_THREADS 128
#endif

struct NbSlot { double x, y, z, r2; };

KF_DEV void sample_point(const double *xi, double r_off_i, const double *q, double &px, double &py,
                         double &pz) {
    px = xadd(xi[0], xmul(r_off_i, q[0]));
    py = xadd(xi[1], xmul(r_off_i, q[1]));
    pz = xadd(xi[2], xmul(r_off_i, q[2]));
}

KF_DEV bool covers(double px, double py, double pz, const NbSlot &s) {
    return d2_rowsum(xsub(px, s.x), xsub(py, s.y), xsub(pz, s.z)) <= s.r2;
}
KF_DEV bool covers_shifted(double px, double py, double pz, const NbSlot &s, int axis, double dr) {
    const double sx = axis == 0 ? xadd(s.x, dr) : s.x;
    const double sy = axis == 1 ? xadd(s.y, dr) : s.y;
    const double sz = axis == 2 ? xadd(s.z, dr) : s.z;
    return d2_rowsum(xsub(px, sx), xsub(py, sy), xsub(pz, sz)) <= s.r2;
}

// Staged neighbour set of one atom (shared memory): coordinates + R_off^2,
// an fp32 spherical-cap prefilter per neighbour, and a largest-cap-first order.
//
// Cap prefilter: for a sample p = r_i + R_i q (|q| = 1) and a neighbour at
// distance d in direction u, |p - r_j|^2 = R_i^2 + d^2 - 2 R_i d (q.u), so j can
// cover p only if q.u >= c1 = (R_i^2 + d^2 - R_j^2) / (2 R_i d), and j displaced
// by dr only if q.u >= c2 = (R_i^2 + d^2 - (R_j + dr)^2) / (2 R_i d).  The fp32
// test q.u >= c - 1e-3 is a strict superset (all rounding is ~1e-7); every
// sample that passes gets the exact fp64 test of the reference.
struct NbSet {
    NbSlot *nb;
    float4 *cap;          // u.x, u.y, u.z, c1
    float *c2;
    unsigned short *ord;  // nearest first
    int32_t *atom;
    double *key;          // sort scratch
};

constexpr float CAP_MARGIN = 1e-3f;

KF_DEV void prepare_neighbors(const double *xi, double r_i, int count, double dr, const NbSet &S) {
    const int P = count <= 1 ? 1 : 1 << (32 - __clz(count - 1));
    for (int m = threadIdx.x; m < P; m += blockDim.x) {
        if (m < count) {
            const NbSlot q = S.nb[m];
            const double dx = q.x - xi[0], dy = q.y - xi[1], dz = q.z - xi[2];
            const double d2 = dx * dx + dy * dy + dz * dz;
            const double d = sqrt(d2);
            const double rj = sqrt(q.r2);
            float4 cp;
            float c2 = -3.f;
            if (d > 1e-6) {
                const double inv = 1.0 / d;
                const double c1 = (r_i * r_i + d2 - q.r2) / (2.0 * r_i * d);
                c2 = (float)((r_i * r_i + d2 - (rj + dr) * (rj + dr)) / (2.0 * r_i * d)) - CAP_MARGIN;
                cp = make_float4((float)(dx * inv), (float)(dy * inv), (float)(dz * inv), (float)c1 - CAP_MARGIN);
            } else {
                cp = make_float4(0.f, 0.f, 0.f, -3.f);
            }
            S.cap[m] = cp;
            S.c2[m] = c2;
            S.key[m] = (double)cp.w;   // largest cap first
        } else {
            S.key[m] = INFINITY;
        }
        S.ord[m] = (unsigned short)m;
    }
    __syncthreads();
    // bitonic sort of (key, ord) ascending
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < P; t += blockDim.x) {
                const int u = t ^ stride;
                if (u > t) {
                    const bool up = (t & size) == 0;
                    const double a = S.key[t], b = S.key[u];
                    if ((a > b) == up) {
                        S.key[t] = b; S.key[u] = a;
                        const unsigned short o = S.ord[t];
                        S.ord[t] = S.ord[u]; S.ord[u] = o;
                    }
                }
            }
            __syncthreads();
        }
}

// States + (optionally) forward-difference events of atom i's samples against
// the staged set; returns this thread's count of covered samples.
//
// Phase A (thread per sample): the neighbours are sorted largest-cap first, so
// most buried samples meet two coverers within the first few; a sample that
// does within QUICK neighbours is state 2 (clamped count, no forces).  The rest
// (exposed, critical, or slow) go to a shared list.
// Phase B (thread per listed sample): the full scan with the clamp at 2, the
// unique coverer, and the forward-difference events; compaction gives each
// warp samples of similar cost.  Both phases use the reference's exact
// coverage arithmetic, so states and forces are bit-identical.
constexpr int QUICK = 8;
constexpr int UND_CAP = 1024;

template <bool WITH_FORCES>
KF_DEV int enumerate_samples(const double *xi, double r_off_i, const double *samples, int N,
                             const NbSet &S, int nn, long long wi, double dr, long long *acc_nb,
                             long long *acc_i, uint8_t *counts_out, int32_t *crit_out) {
    __shared__ int und[UND_CAP];
    __shared__ int n_und;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int quick = min(nn, QUICK);
    int covered = 0;
    for (int k0 = 0; k0 < N; k0 += UND_CAP) {
        const int kend = min(N, k0 + UND_CAP);
        if (threadIdx.x == 0) n_und = 0;
        __syncthreads();
        // ---- phase A
        for (int k = k0 + threadIdx.x; k < kend; k += blockDim.x) {
            const double *q = samples + 3 * k;
            const float qx = (float)q[0], qy = (float)q[1], qz = (float)q[2];
            double px, py, pz;
            sample_point(xi, r_off_i, q, px, py, pz);
            int cnt = 0;
            for (int r = 0; r < quick && cnt < 2; ++r) {
                const int m = S.ord[r];
                const float4 cp = S.cap[m];
                if (qx * cp.x + qy * cp.y + qz * cp.z < cp.w) continue;
                cnt += covers(px, py, pz, S.nb[m]);
            }
            if (cnt >= 2) {
                ++covered;
                if (counts_out) { counts_out[k] = 2; crit_out[k] = -1; }
            } else {
                und[atomicAdd(&n_und, 1)] = k;
            }
        }
        __syncthreads();
        // ---- phase B: thread per listed sample (similar work per warp after compaction)
        const int nu = n_und;
        for (int u = threadIdx.x; u < nu; u += blockDim.x) {
            const int k = und[u];
            const double *q = samples + 3 * k;
            const float qx = (float)q[0], qy = (float)q[1], qz = (float)q[2];
            double px, py, pz;
            sample_point(xi, r_off_i, q, px, py, pz);
            int cnt = 0, crit = -1;
            for (int r = 0; r < nn; ++r) {
                const int m = S.ord[r];
                const float4 cp = S.cap[m];
                if (qx * cp.x + qy * cp.y + qz * cp.z < cp.w) continue;
                if (covers(px, py, pz, S.nb[m])) {
                    crit = m;
                    if (++cnt == 2) break;
                }
            }
            covered += cnt > 0;
            if (counts_out) {
                counts_out[k] = (uint8_t)cnt;
                crit_out[k] = cnt == 1 ? S.atom[crit] : -1;
            }
            if (WITH_FORCES && wi != 0) {
                if (cnt == 0) {
                    // exposed: every neighbour displaced along each axis (solvation.py:224-235)
                    for (int m = 0; m < nn; ++m) {
                        const float4 cp = S.cap[m];
                        if (qx * cp.x + qy * cp.y + qz * cp.z < S.c2[m]) continue;
                        const NbSlot nbm = S.nb[m];
                        for (int s = 0; s < 3; ++s) {
                            if (covers_shifted(px, py, pz, nbm, s, dr)) {
                                atomicAdd(reinterpret_cast<unsigned long long *>(&acc_nb[3 * m + s]),
                                          (unsigned long long)wi);
                                acc_i[s] -= wi;
                            }
                        }
                    }
                } else if (cnt == 1) {
                    // critical: only the recorded coverer, displaced (solvation.py:236-245)
                    for (int s = 0; s < 3; ++s) {
                        if (!covers_shifted(px, py, pz, S.nb[crit], s, dr)) {
                            acc_i[s] += wi;
                            atomicAdd(reinterpret_cast<unsigned long long *>(&acc_nb[3 * crit + s]),
                                      (unsigned long long)(-wi));
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
    return covered;
}

// shared-memory carve-up: nb | cap | acc (also the sort keys) | c2 | atom | ord
KF_DEV NbSet carve(unsigned char *smem, int cap, long long **acc) {
    NbSet S;
    S.nb = reinterpret_cast<NbSlot *>(smem);
    S.cap = reinterpret_cast<float4 *>(S.nb + cap);
    *acc = reinterpret_cast<long long *>(S.cap + cap);
    S.key = reinterpret_cast<double *>(*acc);
    S.c2 = reinterpret_cast<float *>(*acc + 3 * cap);
    S.atom = reinterpret_cast<int32_t *>(S.c2 + cap);
    S.ord = reinterpret_cast<unsigned short *>(S.atom + cap);
    return S;
}

size_t set_smem(int cap) {
    const int P = cap <= 1 ? 1 : 1 << (32 - __builtin_clz(cap - 1));
    return (size_t)P * (sizeof(NbSlot) + sizeof(float4) + 3 * sizeof(long long) + sizeof(float) +
                        sizeof(int32_t) + sizeof(unsigned short));
}

// ---- hot path ---------------------------------------------------------------
//
// Sample groups: the host orders the N sample directions into G groups of (at
// most) 32 that are compact on the sphere (recursive bisection), each with a
// bounding cone (axis a_g, half-angle alpha_g).  A neighbour whose enlarged cap
// (q.u >= c2, which contains the plain cap c1) misses a group's cone can neither
// cover nor, displaced by dr, newly cover any of its samples, so each group
// only visits the neighbours in its candidate bitmask.  One warp owns one group
// at a time, lane = sample: every lane walks the same candidate list (largest
// caps first), so the loop is warp-uniform and the warp leaves as soon as all
// its samples are covered twice.  Coverage and force arithmetic are the
// reference's fp64 operations (see above); results are bit-identical.
struct GroupSmem {
    NbSlot *nb;        // [cap] sorted: largest cap first
    float4 *cap;       // [cap] u, c1 - margin
    float *c2;         // [cap] c2 - margin
    int32_t *atom;     // [cap]
    float4 *cone;      // [cap] cos / sin of the enlarged cap, cos / sin of the tightened plain cap
    // staging (aliases acc + masks): unsorted neighbours and their sort keys
    NbSlot *tmp;
    int32_t *tmp_atom;
    float *key;
    long long *acc;    // [3 cap] neighbour-side fixed-point events
    uint32_t *mask;    // [G][cap / 32] candidate bitmasks
    uint32_t *full;    // [G][cap / 32] neighbours covering every sample of the group
};

KF_DEV GroupSmem carve_group(unsigned char *smem, int cap, int G) {
    GroupSmem S;
    S.nb = reinterpret_cast<NbSlot *>(smem);
    S.cap = reinterpret_cast<float4 *>(S.nb + cap);
    S.c2 = reinterpret_cast<float *>(S.cap + cap);
    S.atom = reinterpret_cast<int32_t *>(S.c2 + cap);
    S.cone = reinterpret_cast<float4 *>(S.atom + ((cap + 3) & ~3));
    unsigned char *r1 = reinterpret_cast<unsigned char *>(S.cone + cap);
    S.tmp = reinterpret_cast<NbSlot *>(r1);
    S.tmp_atom = reinterpret_cast<int32_t *>(S.tmp + cap);
    S.key = reinterpret_cast<float *>(S.tmp_atom + cap);
    S.acc = reinterpret_cast<long long *>(r1);
    S.mask = reinterpret_cast<uint32_t *>(S.acc + 3 * cap);
    S.full = S.mask + (size_t)G * ((cap + 31) / 32);
    return S;
}

size_t group_smem(int cap, int G) {
    const size_t base = (size_t)cap * (sizeof(NbSlot) + 2 * sizeof(float4) + sizeof(float)) +
                        (size_t)((cap + 3) & ~3) * sizeof(int32_t);
    const size_t stage = (size_t)cap * (sizeof(NbSlot) + sizeof(int32_t) + sizeof(float));
    const size_t work = (size_t)cap * 3 * sizeof(long long) + 2 * (size_t)G * ((cap + 31) / 32) * sizeof(uint32_t);
    return base + (stage > work ? stage : work);
}

struct SolvArgs {
    int n;
    const double *pos_all;
    const unsigned long long *keys;
    const int32_t *cnt, *start, *atom_slot;
    const double4 *s_pos;
    const int4 *s_aux;
    const float4 *cell_box;   // [B][H][2] members' box (fp32 offsets from the cell centre)
    long long *solv_acc;
    double *cav_atom, *f_exp_out, *a_exp_out;
    kf_status_t *status;
    int32_t *ovf;          // [0]: count, then (b, i) pairs of atoms over the fast capacity
    int ovf_cap;
    int fast_cap;          // primary-pass capacity (<= the build's CAP; tests lower it)
};

// One atom (the whole CTA).  nb_cap = staged-neighbour capacity of this launch;
// OVERFLOW = false: a larger count defers the atom to the overflow list;
// OVERFLOW = true: the large-capacity pass (a larger count is an error).
template <bool OVERFLOW>
KF_DEV void solv_atom(const kf_field_t &f, const SolvArgs &A, int b, int i, int nb_cap) {
    const int n = A.n;
    const double *__restrict__ pos_all = A.pos_all;
    const unsigned long long *__restrict__ keys = A.keys;
    const int32_t *__restrict__ cnt = A.cnt, *__restrict__ start = A.start, *__restrict__ atom_slot = A.atom_slot;
    const double4 *__restrict__ s_pos = A.s_pos;
    const int4 *__restrict__ s_aux = A.s_aux;
    kf_status_t *status = A.status;
    if (status[b].done) return;
    extern __shared__ __align__(16) unsigned char smem[];
    const GroupSmem S = carve_group(smem, nb_cap, f.n_groups);
    __shared__ int nn, next_group, covered_s;
    __shared__ long long acc_i_s[3];
    __shared__ int gfull_s[SOLV_MAX_GROUPS];   // full coverers per sample group
    __shared__ int gf0_s[SOLV_MAX_GROUPS];     // the lowest-index full coverer per sample group
    if (threadIdx.x == 0) { nn = 0; next_group = 0; covered_s = 0; acc_i_s[0] = acc_i_s[1] = acc_i_s[2] = 0; }
    for (int q = threadIdx.x; q < SOLV_MAX_GROUPS; q += blockDim.x) { gfull_s[q] = 0; gf0_s[q] = 0x7fffffff; }
    __syncthreads();

    const size_t ai = (size_t)b * n + i;
    const double xi[3] = {pos_all[3 * ai], pos_all[3 * ai + 1], pos_all[3 * ai + 2]};
    const double r_i = f.r_off[i];
    const uint32_t H = 1u << f.hash_bits;
    const size_t hb = (size_t)b * H, nbase = (size_t)b * n;
    int cx, cy, cz;
    unpack_cell((long long)keys[hb + atom_slot[ai]], cx, cy, cz);

    // ---- gather the reachable neighbours (stencil cells probed by one warp,
    // their members swept by the whole block) into the staging area
    __shared__ int cell_first[32], cell_pre[33];
    if (threadIdx.x < 32) {
        int first = 0, len = 0;
        if ((int)threadIdx.x < f.n_stencil) {
            const int s = threadIdx.x;
            const int js = cell_probe(keys + hb, H, cx + f.stencil[3 * s], cy + f.stencil[3 * s + 1],
                                      cz + f.stencil[3 * s + 2]);
            if (js >= 0) {
                // skip the cell unless its members' box is within R_off_i + max R_off + pad
                const int nx = cx + f.stencil[3 * s], ny = cy + f.stencil[3 * s + 1], nz = cz + f.stencil[3 * s + 2];
                const float px = (float)(xi[0] - ((double)nx + 0.5) * f.cell);
                const float py = (float)(xi[1] - ((double)ny + 0.5) * f.cell);
                const float pz = (float)(xi[2] - ((double)nz + 0.5) * f.cell);
                const float4 lo = A.cell_box[2 * (hb + js)], hi = A.cell_box[2 * (hb + js) + 1];
                const float gx = fmaxf(fmaxf(lo.x - px, px - hi.x), 0.f);
                const float gy = fmaxf(fmaxf(lo.y - py, py - hi.y), 0.f);
                const float gz = fmaxf(fmaxf(lo.z - pz, pz - hi.z), 0.f);
                const float reach = (float)(r_i + f.r_off_max + f.reach_pad) + 1e-3f;
                if (gx * gx + gy * gy + gz * gz <= reach * reach) { first = start[hb + js]; len = cnt[hb + js]; }
            }
        }
        cell_first[threadIdx.x] = first;
        int incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)threadIdx.x >= o) incl += v;
        }
        cell_pre[threadIdx.x + 1] = incl;
        if (threadIdx.x == 0) cell_pre[0] = 0;
    }
    __syncthreads();
    const int cand = cell_pre[32];
    constexpr int GATHER_UNROLL = 4;   // candidates in flight per thread (independent loads)
    const float r_i_f = (float)r_i;
    for (int c0 = threadIdx.x; c0 < cand; c0 += GATHER_UNROLL * blockDim.x) {
        double4 pjs[GATHER_UNROLL];
        int js[GATHER_UNROLL];
#pragma unroll
        for (int u = 0; u < GATHER_UNROLL; ++u) {
            const int c = c0 + u * blockDim.x;
            js[u] = -1;
            if (c < cand) {
                int lo = 0, hi = 32;
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (cell_pre[mid] <= c) lo = mid; else hi = mid;
                }
                const int kk = cell_first[lo] + (c - cell_pre[lo]);
                pjs[u] = s_pos[nbase + kk];
                js[u] = s_aux[nbase + kk].x;
            }
        }
#pragma unroll
        for (int u = 0; u < GATHER_UNROLL; ++u) {
            const int j = js[u];
            if (j < 0 || j == i) continue;
            const double4 pj = pjs[u];
            const double dx = xi[0] - pj.x, dy = xi[1] - pj.y, dz = xi[2] - pj.z;
            const double lim = r_i + pj.w + f.reach_pad;           // pj.w = R_off_j
            const double d2 = dx * dx + dy * dy + dz * dz;
            if (d2 > lim * lim) continue;
            const int slot = atomicAdd(&nn, 1);
            if (slot < nb_cap) {
                const double r2j = xmul(pj.w, pj.w);                 // = r_off2[j] (host R_off * R_off)
                S.tmp[slot] = NbSlot{pj.x, pj.y, pj.z, r2j};
                S.tmp_atom[slot] = j;
                // sort key c1 (smaller = larger cap, fp32: ordering only); -3 for a coincident atom.
                // The visiting order only decides how soon a walk can stop (states, the unique
                // coverer and the event sums do not depend on it), so the key is c1 mapped to an
                // order-preserving integer, cut to its top 19 bits in bits 12-30, with the slot in
                // the low 12: unique keys below 2^31, so the rank sort counts smaller keys by the
                // sign of a difference (a subtract and a shifted add per pair)
                const float d2f = (float)d2, df = sqrtf(d2f);
                const float kf = d2f > 1e-12f ? (r_i_f * r_i_f + d2f - (float)r2j) / (2.f * r_i_f * df) : -3.f;
                unsigned ku = __float_as_uint(kf);
                ku = (ku & 0x80000000u) ? ~ku : (ku | 0x80000000u);
                reinterpret_cast<unsigned *>(S.key)[slot] = ((ku >> 1) & 0x7ffff000u) | (unsigned)slot;
            }
        }
    }
    __syncthreads();
    const int count = nn;
    if (count > nb_cap) {
        if (threadIdx.x == 0) {
            const int e = OVERFLOW ? A.ovf_cap : atomicAdd(A.ovf, 1);
            if (e < A.ovf_cap) {
                A.ovf[1 + 2 * e] = b;
                A.ovf[2 + 2 * e] = i;
            } else {
                atomicMax(&status[b].overflow, count);
                if (atomicCAS(&status[b].error, KF_ERR_NONE, KF_ERR_CAPACITY) == KF_ERR_NONE)
                    status[b].err_iter = status[b].iter;
            }
        }
        return;
    }
    // ---- rank sort (largest cap first; unique integer keys) and the caps in sorted order
    const double dr = f.delta_r;
    const float drf = (float)dr;
    const unsigned *ukey = reinterpret_cast<const unsigned *>(S.key);
    for (int m = threadIdx.x; m < count; m += blockDim.x) {
        const unsigned km = ukey[m];
        int r = 0;
        for (int t = 0; t < count; ++t) r += (ukey[t] - km) >> 31;   // keys < 2^31: the sign of the difference
        const NbSlot q = S.tmp[m];
        S.nb[r] = q;
        S.atom[r] = S.tmp_atom[m];
        // caps in fp32: prefilters with a 1e-3 margin (fp32 error here ~1e-6)
        const float dx = (float)(q.x - xi[0]), dy = (float)(q.y - xi[1]), dz = (float)(q.z - xi[2]);
        const float d2 = dx * dx + dy * dy + dz * dz;
        if (d2 > 1e-12f) {
            const float d = sqrtf(d2), inv = 1.f / d, r2j = (float)q.r2, rj = sqrtf(r2j);
            const float ri2 = r_i_f * r_i_f, den = 1.f / (2.f * r_i_f * d);
            const float c1 = (ri2 + d2 - r2j) * den - CAP_MARGIN, c2 = (ri2 + d2 - (rj + drf) * (rj + drf)) * den - CAP_MARGIN;
            S.cap[r] = make_float4(dx * inv, dy * inv, dz * inv, c1);
            S.c2[r] = c2;
            // the mask pass's cone terms: enlarged cap (cos, sin), plain cap tightened
            // by 1e-3 (c1 is c1 - 1e-3 already) for the full-cover test
            const float cb = fminf(fmaxf(c2, -1.f), 1.f), sb = sqrtf(fmaxf(0.f, 1.f - cb * cb));
            float cf = 2.f, sf = 0.f;
            if (c1 > -2.f) {
                cf = c1 + 2e-3f;
                sf = sqrtf(fmaxf(0.f, 1.f - cf * cf));
            }
            S.cone[r] = make_float4(cb, sb, cf, sf);
        } else {
            S.cap[r] = make_float4(0.f, 0.f, 0.f, -3.f);
            S.c2[r] = -3.f;
            S.cone[r] = make_float4(-1.f, 0.f, 2.f, 0.f);   // keep (cb <= -cos alpha), never full
        }
    }
    __syncthreads();
    // ---- candidate bitmasks: group cone vs enlarged cap
    const int G = f.n_groups, W = (count + 31) >> 5;
    if (G <= 32) {
        // lane = sample group (its cone in registers), each warp builds whole
        // 32-neighbour words, the neighbours' cap terms broadcast from shared memory
        const int lane = threadIdx.x & 31, g = lane;
        const bool gl = g < G;
        const float4 ax = gl ? reinterpret_cast<const float4 *>(f.grp_cone)[2 * g] : make_float4(0.f, 0.f, 0.f, 2.f);
        const float sin_a = gl ? f.grp_cone[8 * g + 4] : 0.f;
        for (int w = threadIdx.x >> 5; w < W; w += blockDim.x >> 5) {
            const int m0 = w << 5, mn = min(32, count - m0);
            uint32_t bits = 0u, fbits = 0u;
            // neighbours in reverse order, each bit shifted in from the bottom (bit t ends at
            // position t); both tests evaluated without short-circuit (no predicated chains)
#pragma unroll 4
            for (int t = mn - 1; t >= 0; --t) {
                const float4 cp = S.cap[m0 + t], cn = S.cone[m0 + t];
                const float dot = ax.x * cp.x + ax.y * cp.y + ax.z * cp.z;
                // cone (a_g, alpha) meets the enlarged cap (u, beta): angle(a, u) <= alpha + beta
                const bool keep = (cn.x <= -ax.w) | (dot >= ax.w * cn.x - sin_a * cn.y - 1e-3f);
                // cone inside the tightened plain cap (beta1 > alpha, angle(a, u) <= beta1 - alpha):
                // every sample of the group is covered by m, exactly (margins >> rounding)
                const bool full = (cn.z < ax.w) & (dot >= ax.w * cn.z + sin_a * cn.w + 1e-3f);
                bits = (bits << 1) | (uint32_t)keep;
                fbits = (fbits << 1) | (uint32_t)full;
            }
            if (gl) {
                S.mask[g * W + w] = bits; S.full[g * W + w] = fbits;
                if (fbits && g < SOLV_MAX_GROUPS) {
                    atomicAdd(&gfull_s[g], __popc(fbits));
                    atomicMin(&gf0_s[g], (w << 5) + __ffs(fbits) - 1);
                }
            }
        }
    } else {
        // lane = neighbour of word w (its cap in registers), warps sweep the groups
        const int lane = threadIdx.x & 31;
        for (int w = 0; w < W; ++w) {
            const int m = (w << 5) + lane;
            float4 cp = make_float4(0.f, 0.f, 0.f, 0.f), cn = make_float4(1.f, 0.f, 2.f, 0.f);
            const bool live = m < count;
            if (live) { cp = S.cap[m]; cn = S.cone[m]; }
            for (int g = threadIdx.x >> 5; g < G; g += blockDim.x >> 5) {
                const float4 ax = reinterpret_cast<const float4 *>(f.grp_cone)[2 * g];
                const float sin_a = f.grp_cone[8 * g + 4];
                const float dot = ax.x * cp.x + ax.y * cp.y + ax.z * cp.z;
                const bool keep = live && (cn.x <= -ax.w || dot >= ax.w * cn.x - sin_a * cn.y - 1e-3f);
                const bool full = live && cn.z < ax.w && dot >= ax.w * cn.z + sin_a * cn.w + 1e-3f;
                const uint32_t bits = __ballot_sync(0xffffffffu, keep);
                const uint32_t fbits = __ballot_sync(0xffffffffu, full);
                if (lane == 0) {
                    S.mask[g * W + w] = bits; S.full[g * W + w] = fbits;
                    if (fbits && g < SOLV_MAX_GROUPS) {
                        atomicAdd(&gfull_s[g], __popc(fbits));
                        atomicMin(&gf0_s[g], (w << 5) + __ffs(fbits) - 1);
                    }
                }
            }
        }
    }
    for (int m = threadIdx.x; m < 3 * count; m += blockDim.x) S.acc[m] = 0;
    __syncthreads();
    // groups with two full coverers are settled (every sample covered twice, no
    // events): their samples are counted here and only the open groups are listed
    // for the warps (list order is free: groups are independent, totals integer)
    __shared__ int glist_s[SOLV_MAX_GROUPS];
    __shared__ int n_open_s;
    const bool use_list = G <= SOLV_MAX_GROUPS;
    if (threadIdx.x == 0) n_open_s = 0;
    __syncthreads();
    if (use_list)
        for (int t = threadIdx.x; t < G; t += blockDim.x) {
            if (gfull_s[t] >= 2) atomicAdd(&covered_s, (int)f.grp_cone[8 * t + 5]);
            else glist_s[atomicAdd(&n_open_s, 1)] = t;
        }
    __syncthreads();
    const int n_open = use_list ? n_open_s : G;

    // ---- one warp per sample group, lane = sample
    const int lane = threadIdx.x & 31;
    const long long wi = f.w_int[i];
    long long acc_i[3] = {0, 0, 0};
    int covered = 0;
    for (;;) {
        // groups are taken from a block counter: warps that meet cheap
        // (buried) groups take more of them
        int k = 0;
        if (lane == 0) k = atomicAdd(&next_group, 1);
        k = __shfl_sync(0xffffffffu, k, 0);
        if (k >= n_open) break;
        const int g = use_list ? glist_s[k] : k;
        const bool valid = lane < (int)f.grp_cone[8 * g + 5];
        const uint32_t *gm = S.mask + g * W, *gf = S.full + g * W;
        // neighbours covering the whole group: two of them settle every sample (counted,
        // with the lowest-index one, in the mask pass when the groups are tracked)
        int nfull = 0, f0 = -1;
        if (use_list) {
            nfull = gfull_s[g];
            f0 = nfull ? gf0_s[g] : -1;
        } else {
            for (int w = 0; w < W; ++w) {
                const uint32_t fb = gf[w];
                if (fb && f0 < 0) f0 = (w << 5) + __ffs(fb) - 1;
                nfull += __popc(fb);
            }
        }
        if (lane == 0) { SSTAT(0, 1); SSTAT(7, W); }
        if (nfull >= 2) {
            if (lane == 0) SSTAT(1, 1);
            if (valid) ++covered;
            continue;
        }
        if (lane == 0 && nfull == 1) SSTAT(2, 1);
        // unsettled group: this lane's sample point
        const double *q = f.samples_grp + 3 * (32 * g + (valid ? lane : 0));
        const float qx = (float)q[0], qy = (float)q[1], qz = (float)q[2];
        double px, py, pz;
        sample_point(xi, r_i, q, px, py, pz);
        int cnt = valid ? nfull : 2, crit = nfull == 1 ? f0 : -1;
        // candidates largest cap first; the warp leaves as soon as every sample is
        // covered twice (a vote after every candidate: C5 water 12.65 ms against 12.84 /
        // 12.92 / 13.15 ms voting every 2 / 4 / 8)
        for (int w = 0; w < W; ++w) {
            uint32_t bits = gm[w] & ~gf[w];
            bool all_done = false;
            while (bits) {
                const int m = (w << 5) + __ffs(bits) - 1;
                bits &= bits - 1u;
                if (lane == 0) SSTAT(3, 1);
                // |p - r_j|^2 = R_i^2 + d^2 - 2 R_i d (q.u), so j covers p iff q.u >= c1
                // exactly; cap.w = c1 - 1e-3.  Outside the +-1e-3 band around c1 the fp32
                // test decides (its error is ~1e-6, and so far from the boundary the
                // reference's fp64 test agrees); inside it, the reference's exact fp64
                // test.  (cap.w = -3: a coincident neighbour, always the exact test.)
                // predicated: every lane computes the fp32 test, lanes already covered
                // twice discard it; the rare exact test behind a warp vote (no divergent
                // branches, so no reconvergence barriers per candidate)
                {
                    const float4 cp = S.cap[m];
                    const float dot = qx * cp.x + qy * cp.y + qz * cp.z;
                    const bool open = cnt < 2;
                    bool cov = open & (dot >= cp.w);
                    const bool ex = cov & ((dot < cp.w + 2.f * CAP_MARGIN) | (cp.w < -2.f));
                    if (__any_sync(0xffffffffu, ex))
                        if (ex) cov = covers(px, py, pz, S.nb[m]);
                    crit = cov ? m : crit;
                    cnt += cov ? 1 : 0;
                }
                if (__all_sync(0xffffffffu, cnt >= 2)) { all_done = true; break; }
            }
            if (all_done || __all_sync(0xffffffffu, cnt >= 2)) break;
        }
        if (valid) covered += cnt > 0;
#ifdef SOLV_STATS
        { const unsigned ex = __ballot_sync(0xffffffffu, valid && cnt == 0), cr = __ballot_sync(0xffffffffu, valid && cnt == 1);
          if (lane == 0) { SSTAT(4, __popc(ex)); SSTAT(5, __popc(cr)); if (ex) SSTAT(6, 1); } }
#endif
        if (wi == 0 || !valid) continue;
        if (cnt == 0) {
            // exposed: every candidate displaced along each axis (solvation.py:224-235)
            for (int w = 0; w < W; ++w) {
                uint32_t bits = gm[w];
                while (bits) {
                    const int m = (w << 5) + __ffs(bits) - 1;
                    bits &= bits - 1u;
                    const float4 cp = S.cap[m];
                    if (qx * cp.x + qy * cp.y + qz * cp.z < S.c2[m]) continue;
                    const NbSlot nbm = S.nb[m];
                    for (int s = 0; s < 3; ++s) {
                        if (covers_shifted(px, py, pz, nbm, s, dr)) {
                            atomicAdd(reinterpret_cast<unsigned long long *>(&S.acc[3 * m + s]),
                                      (unsigned long long)wi);
                            acc_i[s] -= wi;
                        }
                    }
                }
            }
        } else if (cnt == 1) {
            // critical: only the recorded coverer, displaced (solvation.py:236-245)
            const NbSlot nbc = S.nb[crit];
            for (int s = 0; s < 3; ++s) {
                if (!covers_shifted(px, py, pz, nbc, s, dr)) {
                    acc_i[s] += wi;
                    atomicAdd(reinterpret_cast<unsigned long long *>(&S.acc[3 * crit + s]),
                              (unsigned long long)(-wi));
                }
            }
        }
    }
    // integer totals: order-free shared atomics (no block-wide reduction tree)
    const int wcov = __reduce_add_sync(0xffffffffu, covered);
    if (lane == 0 && wcov) atomicAdd(&covered_s, wcov);
    for (int s = 0; s < 3; ++s)
        if (acc_i[s] != 0)
            atomicAdd(reinterpret_cast<unsigned long long *>(&acc_i_s[s]), (unsigned long long)acc_i[s]);
    __syncthreads();
    long long *acc = A.solv_acc + (size_t)b * n * 3;
    for (int m = threadIdx.x; m < 3 * count; m += blockDim.x) {
        const long long v = S.acc[m];
        if (v != 0)
            atomicAdd(reinterpret_cast<unsigned long long *>(&acc[3 * (size_t)S.atom[m / 3] + m % 3]),
                      (unsigned long long)v);
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < 3; ++s)
            if (acc_i_s[s] != 0)
                atomicAdd(reinterpret_cast<unsigned long long *>(&acc[3 * (size_t)i + s]),
                          (unsigned long long)acc_i_s[s]);
        // f_exp = (N - covered) / N; a_exp = f_exp * (4 pi R_off^2); term = gamma * a_exp
        const long long cov = covered_s;
        const double f_exp = (double)(f.n_samples - cov) / (double)f.n_samples;
        const double a_exp = xmul(f_exp, xmul(f.four_pi, f.r_off2[i]));
        A.cav_atom[ai] = xmul(f.gamma[i], a_exp);
        if (A.f_exp_out) { A.f_exp_out[ai] = f_exp; A.a_exp_out[ai] = a_exp; }
    }
}

// Primary pass: one CTA per (trajectory, solvation atom) with a small staging
// capacity CAP (more CTAs per SM); the rare atom with more reachable neighbours
// is deferred to solv_overflow_kernel.  Two builds: ensembles (many small CTAs
// resident, CAP 144) and single chains (CAP 256: denser chains overflow less).
// (MINB 10 for the ensemble build: 48 registers, 60 B of spill stores, as fast as MINB 12 at 40
// registers with 128 B of spills (13.10 vs 13.11 ms per C5 water step); 8 (64 registers) 14.26 ms.)
template <int CAP, int MINB>
__global__ void __launch_bounds__(SOLV_GROUP_THREADS, MINB)
solv_group_kernel(const __grid_constant__ kf_field_t f, const SolvArgs A, int n_solv, const int32_t *__restrict__ solv_atoms) {
    solv_atom<false>(f, A, blockIdx.x / n_solv, solv_atoms[blockIdx.x % n_solv], min(CAP, A.fast_cap));
}
#ifndef SOLV_MINB_ENS
#define SOLV_MINB_ENS 10
#endif
constexpr int SOLV_CAP_ENSEMBLE = 144, SOLV_MINB_ENSEMBLE = SOLV_MINB_ENS;
constexpr int SOLV_CAP_SINGLE = 256, SOLV_MINB_SINGLE = 8;
constexpr int SOLV_ENSEMBLE_MIN_B = 16;
#ifndef OVF_BLOCKS_PER_SM
#define OVF_BLOCKS_PER_SM 4   // resident CTAs per SM of the overflow pass (49 KB of staging each)
#endif

__global__ void __launch_bounds__(SOLV_GROUP_THREADS)
solv_overflow_kernel(const __grid_constant__ kf_field_t f, const SolvArgs A, int nb_cap) {
    const int m = min(*A.ovf, A.ovf_cap);
    for (int e = blockIdx.x; e < m; e += gridDim.x) {
        solv_atom<true>(f, A, A.ovf[1 + 2 * e], A.ovf[2 + 2 * e], nb_cap);
        __syncthreads();
    }
}

// forces += acc * quantum (solvation.py:255; kcm.py:140)
__global__ void solv_combine_kernel(int B, int n, double quantum, const long long *__restrict__ acc,
                                    double *__restrict__ forces, const kf_status_t *status) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (long long)B * n * 3) return;
    const int b = (int)(gid / (3LL * n));
    if (status[b].done) return;
    forces[gid] = xadd(forces[gid], xmul(__ll2double_rn(acc[gid]), quantum));
}

// ---- API path: explicit CSR neighbour lists (B = 1) ---------------------------

KF_DEV int stage_from_list(const double *pos, const double *r_off, const double *r_off2, int i,
                           const int64_t *nb_off, const int64_t *nbl, double pad, NbSlot *nb,
                           int32_t *nb_atom, int nb_cap, int *nn) {
    const double *xi = pos + 3 * (size_t)i;
    for (long long e = nb_off[i] + threadIdx.x; e < nb_off[i + 1]; e += blockDim.x) {
        const int j = (int)nbl[e];
        const double *xj = pos + 3 * (size_t)j;
        const double dx = xi[0] - xj[0], dy = xi[1] - xj[1], dz = xi[2] - xj[2];
        const double lim = r_off[i] + r_off[j] + pad;
        if (dx * dx + dy * dy + dz * dz > lim * lim) continue;
        const int slot = atomicAdd(nn, 1);
        if (slot < nb_cap) { nb[slot] = NbSlot{xj[0], xj[1], xj[2], r_off2[j]}; nb_atom[slot] = j; }
    }
    __syncthreads();
    return *nn;
}

__global__ void __launch_bounds__(SOLV_THREADS)
sasa_api_kernel(const double *__restrict__ pos, const double *__restrict__ r_off,
                const double *__restrict__ r_off2, const double *__restrict__ samples, int N,
                const int64_t *__restrict__ nb_off, const int64_t *__restrict__ nbl, double pad,
                uint8_t *__restrict__ counts, int32_t *__restrict__ critical,
                int64_t *__restrict__ covered, const double *__restrict__ gamma, double four_pi,
                double *__restrict__ f_exp, double *__restrict__ a_exp, double *__restrict__ cav,
                int nb_cap, int *overflow) {
    const int i = blockIdx.x;
    extern __shared__ __align__(16) unsigned char smem[];
    long long *scratch;
    const NbSet S = carve(smem, nb_cap, &scratch);
    __shared__ int nn;
    __shared__ double red[32];
    if (threadIdx.x == 0) nn = 0;
    __syncthreads();
    const int count = stage_from_list(pos, r_off, r_off2, i, nb_off, nbl, pad, S.nb, S.atom, nb_cap, &nn);
    if (count > nb_cap) {
        if (threadIdx.x == 0) atomicMax(overflow, count);
        return;
    }
    const double xi[3] = {pos[3 * (size_t)i], pos[3 * (size_t)i + 1], pos[3 * (size_t)i + 2]};
    prepare_neighbors(xi, r_off[i], count, 0.0, S);
    const bool empty_list = nb_off[i + 1] == nb_off[i];
    const int cov = enumerate_samples<false>(xi, r_off[i], samples, N, S, count, 0, 0.0, nullptr,
                                             nullptr, counts + (size_t)i * N, critical + (size_t)i * N);
    const double total = block_sum((double)cov, red);
    if (threadIdx.x == 0) {
        const int64_t c = empty_list ? 0 : (int64_t)total;
        covered[i] = c;
        // f_exp = (nq - covered) / float(nq); a_exp = f_exp * (4 pi * r_off2) (solvation.py:177-180)
        const double fe = (double)(N - c) / (double)N;
        const double ae = xmul(fe, xmul(four_pi, r_off2[i]));
        f_exp[i] = fe; a_exp[i] = ae; cav[i] = xmul(gamma[i], ae);
    }
}

__global__ void __launch_bounds__(SOLV_THREADS)
solv_forces_api_kernel(const double *__restrict__ pos, const double *__restrict__ r_off,
                       const double *__restrict__ r_off2, const int64_t *__restrict__ w_int,
                       const double *__restrict__ samples, int N, const int64_t *__restrict__ nb_off,
                       const int64_t *__restrict__ nbl, const uint8_t *__restrict__ counts,
                       const int32_t *__restrict__ critical, double dr, double pad,
                       long long *__restrict__ acc, int nb_cap, int *overflow) {
    const int i = blockIdx.x;
    const long long wi = w_int[i];
    if (wi == 0 || nb_off[i + 1] == nb_off[i]) return;
    extern __shared__ __align__(16) unsigned char smem[];
    long long *acc_nb;
    const NbSet S = carve(smem, nb_cap, &acc_nb);
    NbSlot *nb = S.nb;
    int32_t *nb_atom = S.atom;
    __shared__ int nn;
    __shared__ long long acc_i_s[3];
    if (threadIdx.x == 0) { nn = 0; acc_i_s[0] = acc_i_s[1] = acc_i_s[2] = 0; }
    __syncthreads();
    const int count = stage_from_list(pos, r_off, r_off2, i, nb_off, nbl, pad, nb, nb_atom, nb_cap, &nn);
    if (count > nb_cap) {
        if (threadIdx.x == 0) atomicMax(overflow, count);
        return;
    }
    const double xi[3] = {pos[3 * (size_t)i], pos[3 * (size_t)i + 1], pos[3 * (size_t)i + 2]};
    prepare_neighbors(xi, r_off[i], count, dr, S);
    for (int m = threadIdx.x; m < 3 * count; m += blockDim.x) acc_nb[m] = 0;
    __syncthreads();
    long long acc_i[3] = {0, 0, 0};
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        const int c = counts[(size_t)i * N + k];
        if (c > 1) continue;
        double px, py, pz;
        sample_point(xi, r_off[i], samples + 3 * k, px, py, pz);
        if (c == 0) {
            const float qx = (float)samples[3 * k], qy = (float)samples[3 * k + 1], qz = (float)samples[3 * k + 2];
            for (int m = 0; m < count; ++m) {
                const float4 cp = S.cap[m];
                if (qx * cp.x + qy * cp.y + qz * cp.z < S.c2[m]) continue;
                for (int s = 0; s < 3; ++s)
                    if (covers_shifted(px, py, pz, nb[m], s, dr)) {
                        atomicAdd(reinterpret_cast<unsigned long long *>(&acc_nb[3 * m + s]),
                                  (unsigned long long)wi);
                        acc_i[s] -= wi;
                    }
            }
        } else {
            const int jo = critical[(size_t)i * N + k];
            const NbSlot so{pos[3 * (size_t)jo], pos[3 * (size_t)jo + 1], pos[3 * (size_t)jo + 2], r_off2[jo]};
            for (int s = 0; s < 3; ++s) {
                const double sx = s == 0 ? xadd(so.x, dr) : so.x;
                const double sy = s == 1 ? xadd(so.y, dr) : so.y;
                const double sz = s == 2 ? xadd(so.z, dr) : so.z;
                if (d2_rowsum(xsub(px, sx), xsub(py, sy), xsub(pz, sz)) > so.r2) {
                    acc_i[s] += wi;
                    atomicAdd(reinterpret_cast<unsigned long long *>(&acc[3 * (size_t)jo + s]),
                              (unsigned long long)(-wi));
                }
            }
        }
    }
    for (int s = 0; s < 3; ++s) {
        const long long v = warp_sum_ll(acc_i[s]);
        if ((threadIdx.x & 31) == 0 && v != 0)
            atomicAdd(reinterpret_cast<unsigned long long *>(&acc_i_s[s]), (unsigned long long)v);
    }
    __syncthreads();
    for (int m = threadIdx.x; m < 3 * count; m += blockDim.x) {
        const long long v = acc_nb[m];
        if (v != 0)
            atomicAdd(reinterpret_cast<unsigned long long *>(&acc[3 * (size_t)nb_atom[m / 3] + m % 3]),
                      (unsigned long long)v);
    }
    if (threadIdx.x == 0)
        for (int s = 0; s < 3; ++s)
            if (acc_i_s[s] != 0)
                atomicAdd(reinterpret_cast<unsigned long long *>(&acc[3 * (size_t)i + s]),
                          (unsigned long long)acc_i_s[s]);
}

__global__ void fixed_to_f64_kernel(const long long *acc, int64_t m, double quantum, double *out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) out[k] = xmul(__ll2double_rn(acc[k]), quantum);
}



}  // namespace

int kf_solvation_launch(const kf_field_t *f, kf_batch_t *w, int n, int n_solv, const int32_t *solv_atoms,
                        cudaStream_t s) {
    const int B = w->B;
    KF_CUDA(cudaMemsetAsync(w->solv_acc, 0, sizeof(long long) * (size_t)B * n * 3, s), "memset solv_acc");
    if (n_solv > 0) {
        SolvArgs A;
        A.n = n; A.pos_all = w->pos; A.keys = w->cell_key; A.cnt = w->cell_cnt; A.start = w->cell_start;
        A.atom_slot = w->atom_slot; A.s_pos = reinterpret_cast<const double4 *>(w->s_pos);
        A.s_aux = reinterpret_cast<const int4 *>(w->s_aux); A.solv_acc = w->solv_acc; A.cav_atom = w->cav_atom;
        A.cell_box = reinterpret_cast<const float4 *>(w->cell_box);
        A.f_exp_out = w->f_exp; A.a_exp_out = w->a_exp; A.status = w->status;
        A.ovf = w->solv_ovf; A.ovf_cap = B * n;
        static int fast_cap_env = -1;   // KFB200_SOLV_FAST_CAP: lower the primary capacity (tests)
        if (fast_cap_env < 0) {
            const char *env = getenv("KFB200_SOLV_FAST_CAP");
            fast_cap_env = env ? atoi(env) : 1 << 30;
        }
        A.fast_cap = fast_cap_env;
        // the rank sort packs the staging slot into 12 key bits
        if (w->nb_cap > 4096) KF_CUDA(cudaErrorInvalidValue, "solvation neighbour capacity > 4096");
        KF_CUDA(cudaMemsetAsync(w->solv_ovf, 0, sizeof(int32_t), s), "memset solv_ovf");
        const bool ens = B >= SOLV_ENSEMBLE_MIN_B;
        const int cap = ens ? SOLV_CAP_ENSEMBLE : SOLV_CAP_SINGLE;
        auto kern = ens ? solv_group_kernel<SOLV_CAP_ENSEMBLE, SOLV_MINB_ENSEMBLE>
                        : solv_group_kernel<SOLV_CAP_SINGLE, SOLV_MINB_SINGLE>;
        const size_t smem = group_smem(cap, f->n_groups);
        const size_t smem_ovf = group_smem(w->nb_cap, f->n_groups);
        static size_t opted[2] = {0, 0}, opted_ovf = 0;
        if (smem > opted[ens]) {   // dynamic + static shared memory may pass the 48 KB default
            KF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
            opted[ens] = smem;
        }
        if (smem_ovf > opted_ovf) {
            KF_CUDA(cudaFuncSetAttribute(solv_overflow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem_ovf), "smem attr");
            opted_ovf = smem_ovf;
        }
        kern<<<(unsigned)((long long)B * n_solv), SOLV_GROUP_THREADS, smem, s>>>(*f, A, n_solv, solv_atoms);
        KF_LAUNCH_CHECK("solv_group_kernel");
        static int ovf_grid = 0;
        if (ovf_grid == 0) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&ovf_grid, cudaDevAttrMultiProcessorCount, dev);
            ovf_grid *= OVF_BLOCKS_PER_SM;
        }
        solv_overflow_kernel<<<ovf_grid, SOLV_GROUP_THREADS, smem_ovf, s>>>(*f, A, w->nb_cap);
        KF_LAUNCH_CHECK("solv_overflow_kernel");
    }
    const long long total = (long long)B * n * 3;
    solv_combine_kernel<<<kf_blocks(total, 256), 256, 0, s>>>(B, n, f->quantum, w->solv_acc, w->forces, w->status);
    KF_LAUNCH_CHECK("solv_combine_kernel");
    return 0;
}

int kf_fixed_to_f64_launch(const long long *acc, int64_t m, double quantum, double *out, cudaStream_t s) {
    if (m == 0) return 0;
    fixed_to_f64_kernel<<<kf_blocks(m, 256), 256, 0, s>>>(acc, m, quantum, out);
    KF_LAUNCH_CHECK("fixed_to_f64_kernel");
    return 0;
}

int kf_sasa_api_launch(const double *pos, int n, const double *r_off, const double *r_off2,
                       const double *samples, int N, const int64_t *nb_off, const int64_t *nb, double pad,
                       uint8_t *counts, int32_t *critical, int64_t *covered, const double *gamma,
                       double four_pi, double *f_exp, double *a_exp, double *cav, int nb_cap, int *overflow,
                       cudaStream_t s) {
    if (n == 0) return 0;
    const size_t smem = set_smem(nb_cap);
    if (smem > 48 * 1024)
        KF_CUDA(cudaFuncSetAttribute(sasa_api_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                "smem attr");
    sasa_api_kernel<<<n, SOLV_THREADS, smem, s>>>(pos, r_off, r_off2, samples, N, nb_off, nb, pad, counts,
                                                   critical, covered, gamma, four_pi, f_exp, a_exp, cav,
                                                   nb_cap, overflow);
    KF_LAUNCH_CHECK("sasa_api_kernel");
    return 0;
}

int kf_solv_forces_api_launch(const double *pos, int n, const double *r_off, const double *r_off2,
                              const int64_t *w_int, const double *samples, int N, const int64_t *nb_off,
                              const int64_t *nb, const uint8_t *counts, const int32_t *critical, double dr,
                              double pad, long long *acc, int nb_cap, int *overflow, cudaStream_t s) {
    if (n == 0) return 0;
    const size_t smem = set_smem(nb_cap);
    if (smem > 48 * 1024)
        KF_CUDA(cudaFuncSetAttribute(solv_forces_api_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem), "smem attr");
    solv_forces_api_kernel<<<n, SOLV_THREADS, smem, s>>>(pos, r_off, r_off2, w_int, samples, N, nb_off, nb,
                                                          counts, critical, dr, pad, acc, nb_cap, overflow);
    KF_LAUNCH_CHECK("solv_forces_api_kernel");
    return 0;
}

#ifdef SOLV_STATS
extern "C" int kf_debug_solv_stats(unsigned long long *out) {
    cudaDeviceSynchronize();
    return (int)cudaMemcpyFromSymbol(out, g_solv_stats, sizeof(unsigned long long) * 8);
}
#endif
