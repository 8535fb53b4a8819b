// Cluster-pair elec + vdW kernel for ensembles (K3c): one CTA per trajectory,
// the whole trajectory's pair work on chip.
//
// Reference: Field.evaluate's force phase (/root/reference/pkg/src/kinefold/
// kcm.py:110-127) = extract_pairs (forcefield.py:81-89 -> spatial.py:233-241),
// TreeWeights.weights_for (topology.py:153-195), elec/vdw_pair_quantities
// (forcefield.py:98-113) and the bincount scatter (forcefield.py:162-172).
// The pair SET is the reference's exactly (membership decided as in
// kf_nonbonded.cu: fp32 d^2 outside a 1e-3 A^2 band around each threshold, the
// reference's fp64 einsum-order d^2 inside it), so the grid the reference
// builds (spatial.py:83-230) never needs to exist here: any superset of the
// cut-off pairs gives the same result.
//
// Layout.  Atoms keep the chain's index order, which is spatially compact
// along a polymer: consecutive atoms are bonded or one residue apart.  So no
// binning pass is needed:
//   * j-clusters are octets (atoms 8O..8O+7): each has a centre on a 2^-8 A
//     grid, a half-extent box, and per-atom fp32 offsets from the centre;
//   * i-clusters are quads (atoms 4Q..4Q+3), with the same kind of frame.
// Grid centres make the shift between two frames exact in fp32, so a pair's
// difference vector is (o_i - o_j) + (C_Q - c_O).  Its error is that of the
// fp32 offsets, <= ~1e-6 A.  Pairs closer than 1 A (or inside a cut-off band)
// take the exact fp64 path.
//
// Work.  Each trajectory is one CTA of 16 warps.  Warps take i-quads from a
// shared counter.  Per i-quad, lanes test the box distance to the candidate
// octets O >= Q/2 (half list: every unordered pair once, with j > i inside the
// diagonal octet), 32 octets per ballot.  Each surviving (quad, octet) is one
// warp round of 4 x 8 = 32 pairs, lane = (i of the quad, j of the octet):
//   * the pair math is fp32, branch-free, with predicated selects;
//   * the force on i accumulates in the lane's registers;
//   * the force on j (-f) is summed over the 4 i-lanes by xor shuffles and
//     added to a shared-memory int64 fixed point (2^-28 A units).
// Integer sums are order-free, so the result does not depend on the schedule.
// Vacuum rounds skip the vdW term when the boxes are more than 5 A apart.
// Exact-path pairs add their fp64 forces to the global fixed-point planes
// (fj_add, shared with kf_nonbonded.cu).  The CTA folds those in only if it
// wrote any.
#include "kf_common.cuh"

#include <cooperative_groups.h>

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr double COULOMB_K = 332.06;
constexpr double MIN_DISTANCE = 1e-6;
constexpr float FIXF = 268435456.f;             // 2^28: force fixed point (2^-28 A units)
constexpr double FIX_INV = 1.0 / 268435456.0;
constexpr double FJ_HI = 4096.0, FJ_HI_INV = 1.0 / 4096.0;
constexpr double FJ_LO = 1.0 / 268435456.0, FJ_LO_INV = 268435456.0;
constexpr double FJ_SAT = 4722366482869645213696.0;   // 2^72
constexpr float FAR = 1.0e6f;                   // offset of padding atoms
constexpr double GRID = 256.0;                  // frame centres on a 2^-8 A grid
constexpr double CENTRE_MAX = 32768.0;          // |centre| < 2^15: grid values exact in fp32

struct ClConst {
    float we[4], wv[4];           // weights by class 1..4
    float cut2, cutlo, tv2, te2;  // cut-offs (A^2); cutlo = cut2 - band
    float band, f64_d2;
    float pre2, pre2v;            // box pretests: cut2 + 1e-2, tv2 + 1e-2
    float kap_inv;
    float kwe[4];                 // K w_elec by class
    int uniform, wnz_mask;        // UniformWeights; bit c-1: class c has a nonzero weight
    float mid, half, band_l;      // lean band test: ||d2 - mid| - half| <= band_l (the two distinct thresholds)
    float close4;                 // class-4 close-pair threshold: f64_d2 if class 4 has a weight, else 1e-4
};

// j-side / exact-path accumulation into the global planes [lo | hi | fp64]
// (same planes and units as kf_nonbonded.cu's half list, cleared by the reader).
KF_DEV void cl_fj_add(long long *planes, long long plane, size_t idx, double v) {
    if (v == 0.0) return;
    if (!(fabs(v) < FJ_SAT)) {
        atomicAdd(reinterpret_cast<double *>(planes + 2 * plane + idx), v);
        return;
    }
    const long long hi_u = __double2ll_rn(v * FJ_HI_INV);
    const double rem = v - (double)hi_u * FJ_HI;
    const long long lo_u = __double2ll_rn(rem * FJ_LO_INV);
    if (lo_u) atomicAdd(reinterpret_cast<unsigned long long *>(planes + idx), (unsigned long long)lo_u);
    if (hi_u) atomicAdd(reinterpret_cast<unsigned long long *>(planes + plane + idx), (unsigned long long)hi_u);
}

__device__ __noinline__ int cl_slow_class(const kf_field_t &f, int i, int j) {
    if (!f.tchain[i] || !f.tchain[j] || abs(f.tres[i] - f.tres[j]) > 1) return 4;
    const int pi = f.tparent[i], gpi = f.tgp[i], ggi = f.tggp[i];
    const int pj = f.tparent[j], gpj = f.tgp[j], ggj = f.tggp[j];
    if (pi == j || pj == i) return 1;
    if (gpi == j || gpj == i || (pi >= 0 && pi == pj)) return 2;
    if (ggi == j || ggj == i || (gpi >= 0 && gpi == pj) || (gpj >= 0 && gpj == pi)) return 3;
    return 4;
}

// The reference's pair in fp64 (forcefield.py:98-113 with kcm.py:115-126's
// per-term cut-offs): membership from the einsum-order d^2, clash guard,
// fp64 force into the global planes (+f on i, -f on j).  Returns the counts;
// energies through e[2].
__device__ __forceinline__ int2 cl_exact_pair(const kf_field_t &f, const double *pos, int i, int j, int cls,
                                           long long *planes, long long plane, size_t nb, kf_status_t *st,
                                           double *e) {
    const double dx = xsub(pos[3 * i], pos[3 * j]), dy = xsub(pos[3 * i + 1], pos[3 * j + 1]),
                 dz = xsub(pos[3 * i + 2], pos[3 * j + 2]);
    const double d2 = d2_einsum(dx, dy, dz);
    if (d2 > f.cut_pair2) return make_int2(0, 0);
    const bool ke = d2 <= f.thr_elec2, kv = d2 <= f.thr_vdw2;
    const double d = sqrt(d2);
    if (d < MIN_DISTANCE) {
        atomicMin(&st->dmin_bits, (unsigned long long)__double_as_longlong(d));
        if (atomicCAS(&st->error, KF_ERR_NONE, KF_ERR_CLASH) == KF_ERR_NONE) st->err_iter = st->iter;
        return make_int2(ke, kv);
    }
    const double we = f.uniform_weights ? f.uniform_value : f.w_elec[cls - 1];
    const double wv = f.uniform_weights ? f.uniform_value : f.w_vdw[cls - 1];
    const double inv_d = 1.0 / d;
    double mag = 0.0;
    if (ke) {
        const double num = COULOMB_K * we * f.q[i] * f.q[j];
        const double ee = f.dielectric_const ? num * inv_d / f.kappa : num * inv_d * inv_d;
        e[0] += ee;
        mag += ee * inv_d;
    }
    if (kv) {
        const double eps = sqrt(f.eps[i] * f.eps[j]);
        const double r = (f.R[i] + f.R[j]) * inv_d;
        const double r2 = r * r, r6 = r2 * r2 * r2;
        e[1] += wv * eps * (r6 * r6 - 2.0 * r6);
        mag += 12.0 * wv * eps * (r6 * r6 - r6) * inv_d;
    }
    const double g = mag * inv_d;
    const double fv[3] = {g * dx, g * dy, g * dz};
    for (int q = 0; q < 3; ++q) {
        cl_fj_add(planes, plane, 3 * (nb + i) + q, fv[q]);
        cl_fj_add(planes, plane, 3 * (nb + j) + q, -fv[q]);
    }
    return make_int2(ke, kv);
}

#ifndef CL_LEAN
#define CL_LEAN 1   // lean straight-line visits (off: the general rounds for every unit, A/B)
#endif
#ifndef CL_WARPS_N
#define CL_WARPS_N 16   // measured (lean visits, C5): 16 warps (64 registers) 0.62 ms vs 14 (72) 0.63, 12 (80) 0.65
#endif
#ifndef CL_MINB
#define CL_MINB 2   // CTAs per SM asked of ptxas for trajectories of <= 1536 atoms
#endif
constexpr int CL_WARPS = CL_WARPS_N;

// Shared-memory layout for trajectories of up to NCAP atoms (a compile-time
// capacity, so every section offset is an immediate).
template <int NCAP>
struct ClLayout {
    static constexpr int NO = NCAP / 8, NQ = NCAP / 4;
    static constexpr int OQ = 0;                        // float4 [NCAP]: octet-frame offset xyz, q
    static constexpr int RS = OQ + 16 * NCAP;           // float2 [NCAP]: R, sqrt(eps)
    static constexpr int ACC_LO = RS + 8 * NCAP;        // u32 [3 NCAP]: force fixed point, bits 0-19 (+ carries)
    static constexpr int ACC_MID = ACC_LO + 12 * NCAP;  // u32 [3 NCAP]: bits 20-39 (+ carries)
    static constexpr int ACC_HI = ACC_MID + 12 * NCAP;  // i32 [3 NCAP]: bits 40- (2^-28 A units overall)
    static constexpr int OCT_C = ACC_HI + 12 * NCAP;    // float4 [NO]: octet centre
    static constexpr int OCT_H = OCT_C + 16 * NO;       // float4 [NO]: octet half-extent
    static constexpr int TOTAL = OCT_H + 16 * NO;
};
constexpr int CL_CAPS[] = {512, 1024, 1536, 2048, 2944};
constexpr int CL_NCAPS = 5;

KF_DEV double grid_round(double v) { return rint(v * GRID) * (1.0 / GRID); }

KF_DEV unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

// Exact fixed-point add without returning atomics: v = a 2^40 + b 2^20 + c with
// b, c in [0, 2^20) goes to three 32-bit words by fire-and-forget shared REDs.
// The unsigned low and middle words stay exact for < 4096 adds per element
// (an atom gets one per i-quad reaching its octet plus its own: <= n/4 + 1, and
// shared memory limits the cluster path to n < 3k), the signed top word carries
// |v| < 2^55 (|F| < 2^27 per add).  Integer adds commute: the total is order-free.
template <int NCAP>
KF_DEV void acc_add(unsigned base, int k, long long v) {
    using L = ClLayout<NCAP>;
    const unsigned c = (unsigned)v & 0xfffffu, b = (unsigned)(v >> 20) & 0xfffffu;
    const int a = (int)(v >> 40);
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(base + L::ACC_LO + 4 * k), "r"(c) : "memory");
    if (b) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(base + L::ACC_MID + 4 * k), "r"(b) : "memory");
    if (a) asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(base + L::ACC_HI + 4 * k), "r"(a) : "memory");
}


KF_DEV float4 lds4(unsigned a) {
    float4 v;
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
KF_DEV float2 lds2(unsigned a) {
    float2 v;
    asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
}

// Class of pair (i, j) in a round of quad Q x octet O that may hold a class < 4
// pair: the host-built codes for the 5 octets of the 64-atom window, else the
// bond-tree test for atoms with a partner beyond the window (class_window).
__device__ __noinline__ int near_class(const kf_field_t &f, int Q, int O, int lane, bool live, int i, int j) {
    const int k = O - (Q >> 1);
    if (k <= 4) return 4 - (int)((f.class_codes[5 * Q + k] >> (2 * lane)) & 3ull);
    if (live && f.class_slow[i]) return cl_slow_class(f, i, j);
    return 4;
}

// Half of a unit round: quad Q (i = 4 Q + ii) against octet O (j = 8 O + js), 32
// pairs, with the octet's data (oj, rj) and the frame shift (c_unit - c_O) loaded by
// the caller.  GEN: the octet may hold class < 4 pairs or the quad's own atoms
// (class codes, own-octet test); otherwise every pair is class 4.  Pairs inside a
// threshold band or closer than f64_d2 (nonzero weight) are queued for the exact
// path.  The force on j accumulates in gj (reduced by the caller once per octet).
template <bool DCONST, int NCAP, bool GEN>
KF_DEV void half(const kf_field_t &f, const ClConst &c, const unsigned long long *qcodes, int n, int O, int Q,
                 int i, bool vi, int lane, const float4 &oi, const float2 &ri, const float4 &oj, const float2 &rj,
                 float sx, float sy, float sz, bool vdw_round, bool wnz4, float &fx, float &fy, float &fz,
                 float &gjx, float &gjy, float &gjz, float &ee, float &ev, int &ce, int &cv, unsigned *exq,
                 int exq_cap, int *exq_n) {
    const int j = 8 * O + (lane >> 2);
    const float dx = (oi.x - oj.x) + sx;   // frame shift exact
    const float dy = (oi.y - oj.y) + sy;
    const float dz = (oi.z - oj.z) + sz;
    const float d2 = dx * dx + dy * dy + dz * dz;
    bool live = vi;
    const float qK = (float)COULOMB_K * oi.w;
    float qq = qK * c.we[3] * oj.w, weps = c.wv[3] * ri.y * rj.y;
    bool wnz = wnz4;
    int code = 0;                                    // 4 - class
    if (GEN) {
        if (O == (Q >> 1)) live &= j > i;            // own octet: each pair once
        if (!c.uniform) {
            const int k = O - (Q >> 1);
            if (k <= 4)   // the quad's 5 window codes, staged per warp at the unit's start
                code = (int)((qcodes[k] >> (2 * lane)) & 3ull);
            else if (live && j < n && f.class_slow[i])
                code = 4 - cl_slow_class(f, i, j);   // tree partner beyond the window
            qq = qK * c.we[3 - code] * oj.w;
            weps = c.wv[3 - code] * ri.y * rj.y;
            wnz = (c.wnz_mask >> (3 - code)) & 1;
        }
    }
    // exact path (queued): inside a threshold band, or closer than f64_d2 with a
    // nonzero weight (or at clash range whatever the weight)
    const float dev = fminf(fminf(fabsf(d2 - c.cut2), fabsf(d2 - c.tv2)), fabsf(d2 - c.te2));
    const bool exact = live & ((dev <= c.band) | ((d2 < c.f64_d2) & (wnz | (d2 < 1e-4f))));
    const unsigned em = __ballot_sync(FULL, exact);
    if (em) {
        int base = 0;
        if (lane == __ffs(em) - 1) base = atomicAdd(exq_n, __popc(em));
        base = __shfl_sync(FULL, base, __ffs(em) - 1);
        const int slot = base + __popc(em & ((1u << lane) - 1u));
        if (exact && slot < exq_cap) exq[slot] = (unsigned)i | ((unsigned)j << 12) | ((unsigned)code << 24);
    }
    const bool fast = live & !exact & (d2 < c.cutlo);
    if (!__any_sync(FULL, fast)) return;
    float inv_r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(inv_r) : "f"(d2));
    const float inv_r2 = inv_r * inv_r;
    const bool ke = fast && d2 <= c.te2;
    const float e = DCONST ? qq * c.kap_inv * inv_r : qq * inv_r2;
    float g = ke ? e * inv_r2 : 0.f;
    ee += ke ? e : 0.f;
    ce += ke;
    if (vdw_round) {   // boxes within the vdW reach
        const bool kv = fast && d2 <= c.tv2;
        const float D = ri.x + rj.x;
        const float sr = D * D * inv_r2;
        const float s3 = sr * sr * sr;
        const float s6 = s3 * s3;
        ev += kv ? weps * (s6 - 2.f * s3) : 0.f;
        g = kv ? __fmaf_rn(12.f * weps * (s6 - s3), inv_r2, g) : g;
        cv += kv;
    }
    const float gx = g * dx, gy = g * dy, gz = g * dz;
    fx += gx; fy += gy; fz += gz;
    gjx += gx; gjy += gy; gjz += gz;
}

// The pair phase of trajectory b by one CTA (sm: the ClLayout<NCAP> dynamic
// shared memory).  Also the middle phase of the fused fold iteration below.
// Membership half of a unit round (see half()): difference vector, class, the
// exact-path queue.  Returns the lanes whose pair takes the fp32 path.
struct Prep { float dx, dy, dz, d2, qq, weps; bool fast; };

KF_DEV Prep prep(const kf_field_t &f, const ClConst &c, bool gen, const unsigned long long *qcodes, int n, int O,
                 int Q, int i, bool vi, int lane, const float4 &oi, const float2 &ri, const float4 &oj,
                 const float2 &rj, float sx, float sy, float sz, bool wnz4, unsigned *exq, int exq_cap, int *exq_n) {
    Prep p;
    const int j = 8 * O + (lane >> 2);
    p.dx = (oi.x - oj.x) + sx;   // frame shift exact
    p.dy = (oi.y - oj.y) + sy;
    p.dz = (oi.z - oj.z) + sz;
    p.d2 = p.dx * p.dx + p.dy * p.dy + p.dz * p.dz;
    bool live = vi;
    const float qK = (float)COULOMB_K * oi.w;
    p.qq = qK * c.we[3] * oj.w;
    p.weps = c.wv[3] * ri.y * rj.y;
    bool wnz = wnz4;
    int code = 0;                                    // 4 - class
    if (gen) {
        if (O == (Q >> 1)) live &= j > i;            // own octet: each pair once
        if (!c.uniform) {
            const int k = O - (Q >> 1);
            if (k <= 4)   // the quad's 5 window codes, staged per warp at the unit's start
                code = (int)((qcodes[k] >> (2 * lane)) & 3ull);
            else if (live && j < n && f.class_slow[i])
                code = 4 - cl_slow_class(f, i, j);   // tree partner beyond the window
            p.qq = qK * c.we[3 - code] * oj.w;
            p.weps = c.wv[3 - code] * ri.y * rj.y;
            wnz = (c.wnz_mask >> (3 - code)) & 1;
        }
    }
    const float d2 = p.d2;
    const float dev = fminf(fminf(fabsf(d2 - c.cut2), fabsf(d2 - c.tv2)), fabsf(d2 - c.te2));
    const bool exact = live & ((dev <= c.band) | ((d2 < c.f64_d2) & (wnz | (d2 < 1e-4f))));
    const unsigned em = __ballot_sync(FULL, exact);
    if (em) {
        int base = 0;
        if (lane == __ffs(em) - 1) base = atomicAdd(exq_n, __popc(em));
        base = __shfl_sync(FULL, base, __ffs(em) - 1);
        const int slot = base + __popc(em & ((1u << lane) - 1u));
        if (exact && slot < exq_cap) exq[slot] = (unsigned)i | ((unsigned)j << 12) | ((unsigned)code << 24);
    }
    p.fast = live & !exact & (d2 < c.cutlo);
    return p;
}

// Math half of a unit round for the fp32-path lanes (others add zeros).
template <bool DCONST>
KF_DEV void pair_math(const ClConst &c, const Prep &p, const float2 &ri, const float2 &rj, bool vdw_round,
                      float &fx, float &fy, float &fz, float &gjx, float &gjy, float &gjz, float &ee, float &ev,
                      int &ce, int &cv) {
    float inv_r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(inv_r) : "f"(p.fast ? p.d2 : 1.f));
    const float inv_r2 = inv_r * inv_r;
    const bool ke = p.fast && p.d2 <= c.te2;
    const float e = DCONST ? p.qq * c.kap_inv * inv_r : p.qq * inv_r2;
    float g = ke ? e * inv_r2 : 0.f;
    ee += ke ? e : 0.f;
    ce += ke;
    if (vdw_round) {   // boxes within the vdW reach
        const bool kv = p.fast && p.d2 <= c.tv2;
        const float D = ri.x + rj.x;
        const float sr = D * D * inv_r2;
        const float s3 = sr * sr * sr;
        const float s6 = s3 * s3;
        ev += kv ? p.weps * (s6 - 2.f * s3) : 0.f;
        g = kv ? __fmaf_rn(12.f * p.weps * (s6 - s3), inv_r2, g) : g;
        cv += kv;
    }
    const float gx = g * p.dx, gy = g * p.dy, gz = g * p.dz;
    fx += gx; fy += gy; fz += gz;
    gjx += gx; gjy += gy; gjz += gz;
}

// Both halves of a class-4 unit round at once in packed fp32 (FADD2 / FMUL2 /
// FFMA2: two lanes' worth of arithmetic per issued instruction, same roundings
// as the scalar ops).  .x = quad A, .y = quad B.  Returns false if neither half
// has an fp32-path pair (nothing accumulated).
KF_DEV float2 f2(float a) { return make_float2(a, a); }
KF_DEV float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }

template <bool DCONST>
KF_DEV bool packed_round(const ClConst &c, int n, int O, int iA, int iB, bool vA, bool vB, int lane, float2 oix,
                         float2 oiy, float2 oiz, float2 qKw, float2 Ri, float2 wsi, const float4 &oj,
                         const float2 &rj, float sx, float sy, float sz, bool vdw_round, bool wnz4, float2 &fx,
                         float2 &fy, float2 &fz, float2 &gj_x, float2 &gj_y, float2 &gj_z, float2 &ee, float2 &ev,
                         int &ce, int &cv, unsigned *exq, int exq_cap, int *exq_n) {
    const int j = 8 * O + (lane >> 2);
    const float2 dx = __fadd2_rn(sub2(oix, f2(oj.x)), f2(sx));   // frame shift exact
    const float2 dy = __fadd2_rn(sub2(oiy, f2(oj.y)), f2(sy));
    const float2 dz = __fadd2_rn(sub2(oiz, f2(oj.z)), f2(sz));
    const float2 d2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
    const float2 a1 = sub2(d2, f2(c.cut2)), a2 = sub2(d2, f2(c.tv2)), a3 = sub2(d2, f2(c.te2));
    const float devA = fminf(fminf(fabsf(a1.x), fabsf(a2.x)), fabsf(a3.x));
    const float devB = fminf(fminf(fabsf(a1.y), fabsf(a2.y)), fabsf(a3.y));
    const bool exA = vA & ((devA <= c.band) | ((d2.x < c.f64_d2) & (wnz4 | (d2.x < 1e-4f))));
    const bool exB = vB & ((devB <= c.band) | ((d2.y < c.f64_d2) & (wnz4 | (d2.y < 1e-4f))));
    if (__any_sync(FULL, exA | exB)) {   // rare: queue the exact-path pairs (class 4)
        const unsigned ma = __ballot_sync(FULL, exA), mb = __ballot_sync(FULL, exB);
        int base = 0;
        if (lane == 0) base = atomicAdd(exq_n, __popc(ma) + __popc(mb));
        base = __shfl_sync(FULL, base, 0);
        const int sa = base + __popc(ma & ((1u << lane) - 1u));
        const int sb2 = base + __popc(ma) + __popc(mb & ((1u << lane) - 1u));
        if (exA && sa < exq_cap) exq[sa] = (unsigned)iA | ((unsigned)j << 12);
        if (exB && sb2 < exq_cap) exq[sb2] = (unsigned)iB | ((unsigned)j << 12);
    }
    const bool fA = vA & !exA & (d2.x < c.cutlo), fB = vB & !exB & (d2.y < c.cutlo);
    if (!__any_sync(FULL, fA | fB)) return false;
    float2 inv_r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(inv_r.x) : "f"(fA ? d2.x : 1.f));
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(inv_r.y) : "f"(fB ? d2.y : 1.f));
    const float2 inv_r2 = __fmul2_rn(inv_r, inv_r);
    const bool keA = fA && d2.x <= c.te2, keB = fB && d2.y <= c.te2;
    const float2 qq = __fmul2_rn(qKw, f2(oj.w));
    const float2 e = DCONST ? __fmul2_rn(__fmul2_rn(qq, f2(c.kap_inv)), inv_r) : __fmul2_rn(qq, inv_r2);
    const float2 ge = __fmul2_rn(e, inv_r2);
    float2 g = make_float2(keA ? ge.x : 0.f, keB ? ge.y : 0.f);
    ee = __fadd2_rn(ee, make_float2(keA ? e.x : 0.f, keB ? e.y : 0.f));
    ce += keA + keB;
    if (vdw_round) {   // boxes within the vdW reach
        const bool kvA = fA && d2.x <= c.tv2, kvB = fB && d2.y <= c.tv2;
        const float2 weps = __fmul2_rn(wsi, f2(rj.y));
        const float2 D = __fadd2_rn(Ri, f2(rj.x));
        const float2 sr = __fmul2_rn(__fmul2_rn(D, D), inv_r2);
        const float2 s3 = __fmul2_rn(__fmul2_rn(sr, sr), sr);
        const float2 s6 = __fmul2_rn(s3, s3);
        const float2 evt = __fmul2_rn(weps, __ffma2_rn(f2(-2.f), s3, s6));     // weps (s6 - 2 s3)
        ev = __fadd2_rn(ev, make_float2(kvA ? evt.x : 0.f, kvB ? evt.y : 0.f));
        const float2 gv = __ffma2_rn(__fmul2_rn(__fmul2_rn(f2(12.f), weps), sub2(s6, s3)), inv_r2, g);
        g = make_float2(kvA ? gv.x : g.x, kvB ? gv.y : g.y);
        cv += kvA + kvB;
    }
    const float2 gx = __fmul2_rn(g, dx), gy = __fmul2_rn(g, dy), gz = __fmul2_rn(g, dz);
    fx = __fadd2_rn(fx, gx); fy = __fadd2_rn(fy, gy); fz = __fadd2_rn(fz, gz);
    gj_x = __fadd2_rn(gj_x, gx); gj_y = __fadd2_rn(gj_y, gy); gj_z = __fadd2_rn(gj_z, gz);
    return true;
}

// ---- lean visits: one (unit, octet) visit as straight-line predicated code ----
// A visit is quads A and B of the unit against octet O: 64 pair slots, two per
// lane (lane = (ii, js): i = 4 QA + ii and 4 QB + ii, j = 8 O + js), in packed
// fp32 (.x = quad A, .y = quad B).  Versus the general rounds above: the pair
// masks are folded into the inverse square distances (masked lanes add exact
// zeros, no per-term selects), the two distinct cut-off thresholds are tested
// as one band test (||d2 - mid| - half| <= band), the class weights come from a
// per-lane register of 2-bit codes and a 4-entry shared table, the force on j is
// reduced over the quad lanes by a transpose-reduce (3 shuffles), and the
// fixed-point adds are unconditional.  Only the exact-path queue (pairs in a
// threshold band or closer than f64_d2: rare) is behind a warp-uniform branch;
// whether the vdW term applies (boxes within its reach) is a template argument:
// the sweep visits the octets of each reach class in separate loops.
struct LeanUnit {
    // packed (quad A, quad B) pairs held as 64-bit registers: the packed ops below
    // take them as-is (a float2 held in two scalar registers costs two moves per use)
    unsigned long long ix, iy, iz;   // i offsets in the unit's octet frame
    unsigned long long qk;           // K q_i (class weight applied per visit)
    unsigned long long ri;           // R_i
    unsigned long long se;           // sqrt(eps_i)
    unsigned codes;       // bits 2k..: 4 - class of (iA, j) in window octet U + k; bits 10 + 2k..: iB;
                          // bits 30 / 31: atoms iA / iB exist (one register, not two predicates)
};

// the exact-path queue, read only on the rare path (kept out of the registers)
struct ExQueue { unsigned *q; int cap; int n; };

// two floats as one 64-bit register pair (the packed ops' operand form)
KF_DEV unsigned long long pair_of(float a, float b) {
    unsigned long long v;
    asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(a), "f"(b));
    return v;
}
// packed pair (64-bit register) + / * a broadcast scalar, and * a float2
KF_DEV float2 padd_b(unsigned long long a, float s) {
    float2 r;
    asm("{\n\t.reg .b64 t, d;\n\tmov.b64 t, {%3, %3};\n\tadd.rn.f32x2 d, %2, t;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(r.x), "=f"(r.y) : "l"(a), "f"(s));
    return r;
}
KF_DEV float2 pmul_b(unsigned long long a, float s) {
    float2 r;
    asm("{\n\t.reg .b64 t, d;\n\tmov.b64 t, {%3, %3};\n\tmul.rn.f32x2 d, %2, t;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(r.x), "=f"(r.y) : "l"(a), "f"(s));
    return r;
}
KF_DEV float2 pmul_pp(unsigned long long a, unsigned long long b) {
    float2 r;
    asm("{\n\t.reg .b64 d;\n\tmul.rn.f32x2 d, %2, %3;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(r.x), "=f"(r.y) : "l"(a), "l"(b));
    return r;
}
KF_DEV float2 pmul_p(unsigned long long a, float2 b) {
    float2 r;
    asm("{\n\t.reg .b64 t, d;\n\tmov.b64 t, {%3, %4};\n\tmul.rn.f32x2 d, %2, t;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(r.x), "=f"(r.y) : "l"(a), "f"(b.x), "f"(b.y));
    return r;
}

// EALL: 0 generic; 1 the elec threshold is the pair cut-off (elec >= vdW: every
// fp32-path pair has the elec term); 2 as 1 with the default field's constants
// (9 / 5 A cut-offs, class-4 weights 1, close threshold 1 A^2) as immediates, so
// the visit loop reloads no constants (checked on the host: kf_cluster.cu
// default_constants).
#ifndef CL_PSTAGE
#define CL_PSTAGE 1
#endif
#ifndef CL_VDW_NOVOTE
#define CL_VDW_NOVOTE 1
#endif
template <int EALL> struct KC {
    static constexpr bool D = EALL == 2;
    KF_DEV static float mid(const ClConst &c) { return D ? 53.f : c.mid; }
    KF_DEV static float half(const ClConst &c) { return D ? 28.f : c.half; }
    KF_DEV static float band(const ClConst &c) { return D ? 1e-3f : c.band_l; }
    KF_DEV static float cutlo(const ClConst &c) { return D ? 81.f - 0.95f * 1e-3f : c.cutlo; }
    KF_DEV static float tv2(const ClConst &c) { return D ? 25.f : c.tv2; }
    KF_DEV static float close4(const ClConst &c) { return D ? 1.f : c.close4; }
    KF_DEV static float we4(const ClConst &c) { return D ? 1.f : c.we[3]; }
    KF_DEV static float wv4(const ClConst &c) { return D ? 1.f : c.wv[3]; }
};

template <bool DCONST, int NCAP, int EALL, bool GEN, bool VDW>
KF_DEV void lean_visit(const ClConst &c, const LeanUnit &u, float2 &fx, float2 &fy, float2 &fz, float2 &ee,
                       float2 &ev, int &ce, int &cv, int U, int O, unsigned sb, const float4 &cu, unsigned wtab,
                       ExQueue *xq) {
    using L = ClLayout<NCAP>;
    const int lane = threadIdx.x & 31, ii = lane & 3, js = lane >> 2;
    const int j = 8 * O + js;
    const int iA = 8 * U + ii, iB = iA + 4;
    const float4 oc = lds4(sb + L::OCT_C + 16 * O);
    const float4 oj = lds4(sb + L::OQ + 16 * j);
    const float2 rj = lds2(sb + L::RS + 8 * j);
    // j in the unit's frame (the frame shift cu - oc is exact: grid centres)
    const float jx = oj.x - (cu.x - oc.x), jy = oj.y - (cu.y - oc.y), jz = oj.z - (cu.z - oc.z);
    const float2 dx = padd_b(u.ix, -jx), dy = padd_b(u.iy, -jy), dz = padd_b(u.iz, -jz);
    const float2 d2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
    // padding atoms (past n) sit at -FAR (i) / +FAR (j) offsets: no pair of theirs meets any
    // threshold, so outside the own-octet visit the atom-exists bits need no test
    bool vA = true, vB = true;
    if (GEN) {
        vA = (u.codes >> 30) & 1u;
        vB = (u.codes >> 31) & 1u;
    }
    float2 qq, weps;
    using K = KC<EALL>;
    float closeA = K::close4(c), closeB = K::close4(c);
    int codeA = 0, codeB = 0;
    if (GEN) {
        vA &= j > iA;   // the own octet: each pair once (always true for O > U)
        vB &= j > iB;
        const int k = O - U;
        if (k <= 4) {
            codeA = (int)(u.codes >> (2 * k)) & 3;
            codeB = (int)(u.codes >> (10 + 2 * k)) & 3;
        }
        // the (quad A, quad B) weights and close thresholds of this code pair, as packed
        // operands straight from the 16-entry shared table
        const unsigned e = wtab + 32u * (unsigned)(codeA + 4 * codeB);
        unsigned long long we, wv;
        asm("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(we), "=l"(wv) : "r"(e));
        qq = __fmul2_rn(pmul_pp(u.qk, we), f2(oj.w));
        weps = __fmul2_rn(pmul_pp(u.se, wv), f2(rj.y));
        const float2 cl = lds2(e + 16u);
        closeA = cl.x;
        closeB = cl.y;
    } else {
        qq = pmul_b(u.qk, K::we4(c) * oj.w);
        weps = pmul_b(u.se, K::wv4(c) * rj.y);
    }
    // exact path: inside the band around either threshold, or close (see prep()).  Beyond
    // the vdW reach (box distance^2 > tv2 + 1e-2) no pair is close or near the vdW threshold,
    // and non-vdW visits only exist when the elec threshold is the pair cut-off (mid + half):
    // one band test (for the default field bitwise the same decision: both differences are
    // exact there)
    bool exA, exB;
    if (!VDW && !GEN && EALL) {
        const float2 t = __fadd2_rn(d2, f2(-(K::mid(c) + K::half(c))));
        exA = vA & (fabsf(t.x) <= K::band(c));
        exB = vB & (fabsf(t.y) <= K::band(c));
    } else {
        const float2 t = __fadd2_rn(d2, f2(-K::mid(c)));
        const float bA = fabsf(fabsf(t.x) - K::half(c)), bB = fabsf(fabsf(t.y) - K::half(c));
        exA = vA & ((bA <= K::band(c)) | (d2.x < closeA));
        exB = vB & ((bB <= K::band(c)) | (d2.y < closeB));
    }
    if (__any_sync(FULL, exA | exB)) {   // rare: queue the exact-path pairs
        const unsigned ma = __ballot_sync(FULL, exA), mb = __ballot_sync(FULL, exB);
        int base = 0;
        if (lane == 0) base = atomicAdd(&xq->n, __popc(ma) + __popc(mb));
        base = __shfl_sync(FULL, base, 0);
        const int sa = base + __popc(ma & ((1u << lane) - 1u));
        const int sb2 = base + __popc(ma) + __popc(mb & ((1u << lane) - 1u));
        unsigned *q = xq->q;
        const int cap = xq->cap;
        if (exA && sa < cap) q[sa] = (unsigned)iA | ((unsigned)j << 12) | ((unsigned)codeA << 24);
        if (exB && sb2 < cap) q[sb2] = (unsigned)iB | ((unsigned)j << 12) | ((unsigned)codeB << 24);
    }
    const bool fA = vA & !exA & (d2.x < K::cutlo(c)), fB = vB & !exB & (d2.y < K::cutlo(c));
    // (boxes within the vdW reach almost always hold a pair inside the cut-off: no vote)
    if (!(VDW && CL_VDW_NOVOTE) && !__any_sync(FULL, fA | fB)) return;
    float2 ir;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(ir.x) : "f"(d2.x));
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(ir.y) : "f"(d2.y));
    const float2 ir2 = __fmul2_rn(ir, ir);
    // masks folded into the inverse distances: masked lanes (inf / NaN there) get 0
    const bool keA = EALL ? fA : (fA && d2.x <= c.te2), keB = EALL ? fB : (fB && d2.y <= c.te2);
    float2 g, e;
    if (DCONST) {
        const float2 irm = make_float2(keA ? ir.x : 0.f, keB ? ir.y : 0.f);
        e = __fmul2_rn(__fmul2_rn(qq, f2(c.kap_inv)), irm);
        g = __fmul2_rn(e, __fmul2_rn(irm, irm));
    } else {
        const float2 ir2e = make_float2(keA ? ir2.x : 0.f, keB ? ir2.y : 0.f);
        e = __fmul2_rn(qq, ir2e);
        g = __fmul2_rn(e, ir2e);
    }
    ee = __fadd2_rn(ee, e);
    ce += (int)keA + (int)keB;
    if (VDW) {   // boxes within the vdW reach
        const bool kvA = fA && d2.x <= K::tv2(c), kvB = fB && d2.y <= K::tv2(c);
        const float2 ir2v = make_float2(kvA ? ir2.x : 0.f, kvB ? ir2.y : 0.f);
        const float2 D = padd_b(u.ri, rj.x);
        const float2 sr = __fmul2_rn(__fmul2_rn(D, D), ir2v);
        const float2 s3 = __fmul2_rn(__fmul2_rn(sr, sr), sr);
        const float2 s6 = __fmul2_rn(s3, s3);
        ev = __ffma2_rn(weps, __ffma2_rn(f2(-2.f), s3, s6), ev);                           // weps (s6 - 2 s3)
        g = __ffma2_rn(__fmul2_rn(__fmul2_rn(f2(12.f), weps), __fadd2_rn(s6, __fmul2_rn(f2(-1.f), s3))), ir2v, g);
        cv += (int)kvA + (int)kvB;
    }
    const float2 gx = __fmul2_rn(g, dx), gy = __fmul2_rn(g, dy), gz = __fmul2_rn(g, dz);
    fx = __fadd2_rn(fx, gx); fy = __fadd2_rn(fy, gy); fz = __fadd2_rn(fz, gz);
    // force on j: -(sum over both halves and the 4 quad lanes), transpose-reduced so
    // that lane ii ends with component ii (lane 3 with 0)
    const float sx = gx.x + gx.y, sy = gy.x + gy.y, sz = gz.x + gz.y;
    const bool hi = ii & 2, od = ii & 1;
    float k0 = hi ? sz : sx, k1 = hi ? 0.f : sy;
    const float s0 = hi ? sx : sz, s1 = hi ? sy : 0.f;
    k0 += __shfl_xor_sync(FULL, s0, 2);
    k1 += __shfl_xor_sync(FULL, s1, 2);
    const float snd = od ? k0 : k1;
    float v = od ? k1 : k0;
    v += __shfl_xor_sync(FULL, snd, 1);
    // lane ii = 3 holds exactly 0 and adds it to word 3 j + 3 (x of j + 1, or the
    // first word past the plane): an add of zero changes nothing, and costs less
    // than a predicated branch around the REDs
    const long long q = __float2ll_rn(-v * FIXF);
    const unsigned addr = sb + 4 * (3 * j + ii);
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr + L::ACC_LO), "r"((unsigned)q & 0xfffffu) : "memory");
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr + L::ACC_MID), "r"((unsigned)(q >> 20) & 0xfffffu)
                 : "memory");
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr + L::ACC_HI), "r"((unsigned)(int)(q >> 40)) : "memory");
}

// The lean sweep of unit U: box pretests of 32 candidate octets at a time (against
// the unit's octet box, reloaded from shared memory per block), then one lean
// visit per surviving octet.  Octets of the first block whose bit is set in gen0
// (the own octet and class-window octets holding class < 4 pairs) take the
// general visit; the others are visited in two loops, within the vdW reach and
// beyond it.
template <bool DCONST, int NCAP, int EALL>
KF_DEV void lean_sweep(const ClConst &c, const LeanUnit &lu, float2 &fx, float2 &fy, float2 &fz, float2 &ee,
                       float2 &ev, int &ce, int &cv, int U, int no, unsigned sb, unsigned gen0, unsigned wtab,
                       ExQueue *xq) {
    using L = ClLayout<NCAP>;
    for (int ob = U; ob < no; ob += 32) {
        const float4 cu = lds4(sb + L::OCT_C + 16 * U);
        unsigned cand, vmask;
        {
            const float4 hu = lds4(sb + L::OCT_H + 16 * U);
            const int Oc = ob + (int)(threadIdx.x & 31);
            float bd2 = 3.0e38f;
            if (Oc < no) {
                const float4 oc = lds4(sb + L::OCT_C + 16 * Oc), oh = lds4(sb + L::OCT_H + 16 * Oc);
                const float gx = fmaxf(fabsf(cu.x - oc.x) - (hu.x + oh.x), 0.f);
                const float gy = fmaxf(fabsf(cu.y - oc.y) - (hu.y + oh.y), 0.f);
                const float gz = fmaxf(fabsf(cu.z - oc.z) - (hu.z + oh.z), 0.f);
                bd2 = gx * gx + gy * gy + gz * gz;
            }
            cand = __ballot_sync(FULL, bd2 <= c.pre2);
            vmask = __ballot_sync(FULL, bd2 <= c.pre2v);
        }
        if (ob == U) {
            unsigned g = cand & gen0;
            cand &= ~gen0;
            while (g) {
                const int t = __ffs(g) - 1;
                g &= g - 1u;
                if ((vmask >> t) & 1u)
                    lean_visit<DCONST, NCAP, EALL, true, true>(c, lu, fx, fy, fz, ee, ev, ce, cv, U, ob + t, sb, cu,
                                                               wtab, xq);
                else
                    lean_visit<DCONST, NCAP, EALL, true, false>(c, lu, fx, fy, fz, ee, ev, ce, cv, U, ob + t, sb, cu,
                                                                wtab, xq);
            }
        }
        unsigned m = cand & vmask;
        while (m) {
            const int t = __ffs(m) - 1;
            m &= m - 1u;
            lean_visit<DCONST, NCAP, EALL, false, true>(c, lu, fx, fy, fz, ee, ev, ce, cv, U, ob + t, sb, cu, wtab,
                                                        xq);
        }
        m = cand & ~vmask;
        while (m) {
            const int t = __ffs(m) - 1;
            m &= m - 1u;
            lean_visit<DCONST, NCAP, EALL, false, false>(c, lu, fx, fy, fz, ee, ev, ce, cv, U, ob + t, sb, cu, wtab,
                                                         xq);
        }
    }
}

template <bool DCONST, int NCAP, int EALL>
KF_DEV void cluster_pairs_cta(const kf_field_t &f, const ClConst &c, int n, int b, const double *__restrict__ pos_all,
                              double *__restrict__ forces, double *__restrict__ e_atom,
                              long long *__restrict__ pair_count, kf_status_t *status, long long *__restrict__ planes,
                              unsigned *__restrict__ exq_all, int exq_cap, unsigned char *sm, int nbatch,
                              int split, int rank) {
    using L = ClLayout<NCAP>;
    constexpr int CL_THREADS = CL_WARPS * 32;
    // split > 1: the trajectory's units are shared by the `split` CTAs of a thread-block
    // cluster (rank r takes units r, r + split, ...); each CTA accumulates into its own
    // shared fixed point and the partial sums are combined through distributed shared
    // memory at the end.  Each CTA gets 1 / split of the trajectory's exact-pair queue.
    exq_all += (size_t)b * exq_cap * 2 + (size_t)rank * 2 * (exq_cap / split);
    exq_cap /= split;
    __shared__ int next_q, extent_bad;
    __shared__ ExQueue xq;   // the exact-path queue: scratch pointer, capacity, count
    __shared__ unsigned cnt_e, cnt_v;
    __shared__ double red_e[CL_WARPS][2];
    __shared__ unsigned long long qcodes[CL_WARPS][10];  // the current unit's window class codes (2 quads)
    // lean general visits: by code pair (codeA + 4 codeB): (w_elec A, B, w_vdw A, B), (close A, B, 0, 0)
    __shared__ __align__(16) float4 wpair[16][2];
#if CL_PSTAGE
    __shared__ __align__(8) float2 pstage[CL_WARPS][32];   // lean units: packed-operand staging
#endif
    if (threadIdx.x < 16) {
        const int ca = 3 - (int)(threadIdx.x & 3), cb = 3 - (int)(threadIdx.x >> 2);
        wpair[threadIdx.x][0] = make_float4(c.we[ca], c.we[cb], c.wv[ca], c.wv[cb]);
        wpair[threadIdx.x][1] = make_float4(((c.wnz_mask >> ca) & 1) ? c.f64_d2 : 1e-4f,
                                            ((c.wnz_mask >> cb) & 1) ? c.f64_d2 : 1e-4f, 0.f, 0.f);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int no = (n + 7) / 8, nq = (n + 3) / 4;
    const unsigned base = smem_u32(sm);
    const double *pos = pos_all + 3 * (size_t)b * n;
    const float4 *apar = reinterpret_cast<const float4 *>(f.atom_par);
    // each quad's (elec, vdW) energy goes to e_atom[quad] (global scratch, read back
    // in quad order at the end; the totals then sit at atom 0)
    double *e_q = e_atom + 2 * (size_t)b * n;
    if (threadIdx.x == 0) {
        next_q = CL_WARPS; extent_bad = 0; cnt_e = 0; cnt_v = 0;
        xq.q = exq_all; xq.cap = exq_cap; xq.n = 0;
    }
    // exact-path pairs are queued (packed i | j << 12 | class << 24) into this
    // trajectory's share of a scratch buffer and evaluated after the sweep, in
    // sorted order (deterministic), off the hot loop
    unsigned *exq = exq_all;

    // ---- 1. frames: octet and quad grid centres, half-extent boxes, offsets ----
    for (int a0 = 32 * warp; a0 < 8 * no; a0 += 32 * CL_WARPS) {
        const int a = a0 + lane;
        const bool ok = a < n;
        double x = 0.0, y = 0.0, z = 0.0;
        if (ok) { x = pos[3 * a]; y = pos[3 * a + 1]; z = pos[3 * a + 2]; }
        double lo[3] = {ok ? x : INFINITY, ok ? y : INFINITY, ok ? z : INFINITY};
        double hi[3] = {ok ? x : -INFINITY, ok ? y : -INFINITY, ok ? z : -INFINITY};
        // every octet / quad below no / nq holds at least one atom; lanes past
        // the last one only take part in the shuffles
        const bool in_oct = a < 8 * no;
        bool bad = false;
#pragma unroll
        for (int m = 1; m < 8; m <<= 1) {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                lo[q] = fmin(lo[q], __shfl_xor_sync(FULL, lo[q], m));
                hi[q] = fmax(hi[q], __shfl_xor_sync(FULL, hi[q], m));
            }
        }
        double ctr[3];
        float hx[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            ctr[q] = grid_round(0.5 * (lo[q] + hi[q]));
            hx[q] = __double2float_ru(fmax(hi[q] - ctr[q], ctr[q] - lo[q]));
        }
        bad |= in_oct && !(fabs(ctr[0]) < CENTRE_MAX && fabs(ctr[1]) < CENTRE_MAX && fabs(ctr[2]) < CENTRE_MAX);
        if (bad) extent_bad = 1;
        const float4 par = ok ? apar[a] : make_float4(0.f, 0.f, 0.f, 0.f);
        if (in_oct) {
            reinterpret_cast<float4 *>(sm + L::OQ)[a] =
                ok ? make_float4(__double2float_rn(x - ctr[0]), __double2float_rn(y - ctr[1]),
                                 __double2float_rn(z - ctr[2]), par.x)
                   : make_float4(FAR, FAR, FAR, 0.f);
            reinterpret_cast<float2 *>(sm + L::RS)[a] = make_float2(par.y, par.z);
        }
        if ((lane & 7) == 0 && in_oct) {
            const int O = a >> 3;
            reinterpret_cast<float4 *>(sm + L::OCT_C)[O] = make_float4((float)ctr[0], (float)ctr[1], (float)ctr[2], 0.f);
            reinterpret_cast<float4 *>(sm + L::OCT_H)[O] = make_float4(hx[0], hx[1], hx[2], 0.f);
        }
    }
    for (int k = threadIdx.x; k < 9 * NCAP; k += CL_THREADS)   // the three adjacent word planes
        reinterpret_cast<unsigned *>(sm + L::ACC_LO)[k] = 0u;
    __syncthreads();
    if (extent_bad) {   // centres past 2^15 A: the exact-shift frames do not hold
        if (threadIdx.x == 0 && atomicCAS(&status[b].error, KF_ERR_NONE, KF_ERR_EXTENT) == KF_ERR_NONE)
            status[b].err_iter = status[b].iter;
        return;
    }

    // ---- 2. units of two quads (one i-octet) against candidate octets ---------
    // Unit U = quads 2U and 2U+1 = the atoms of octet U, so both quads share U's
    // frame: per candidate octet O the j data and the frame shift are loaded once,
    // the two quads' rounds run back to back (4 x 8 pairs each), and the force on j
    // is reduced over the quad lanes once per octet.
    // (lane and the shared base are pinned in registers: the compiler would
    // otherwise rematerialise them from special registers in every round)
    int lane_p = lane;
    unsigned sb = base, wsb = smem_u32(wpair);
    asm volatile("" : "+r"(lane_p), "+r"(sb), "+r"(wsb));
    const int ii = lane_p & 3, js = lane_p >> 2;
    const bool wnz4 = (c.wnz_mask >> 3) & 1;          // class 4 has a nonzero weight
    int ce = 0, cv = 0;                               // pair counts: integers, order-free across units
    int U = rank + split * warp;
    while (U < no) {
        const int QA = 2 * U, QB = 2 * U + 1;
        const int iA = 4 * QA + ii, iB = 4 * QB + ii;
        const bool vA = iA < n, vB = iB < n && QB < nq;
        const float4 oiA = vA ? lds4(sb + L::OQ + 16 * iA) : make_float4(-FAR, -FAR, -FAR, 0.f);
        const float4 oiB = vB ? lds4(sb + L::OQ + 16 * iB) : make_float4(-FAR, -FAR, -FAR, 0.f);
        const float2 riA = lds2(sb + L::RS + 8 * (vA ? iA : 0)), riB = lds2(sb + L::RS + 8 * (vB ? iB : 0));
        const float4 cu = lds4(sb + L::OCT_C + 16 * U), hu = lds4(sb + L::OCT_H + 16 * U);
        // this lane's class codes of the unit's window octets, which of those octets
        // hold class < 4 pairs, and whether the unit has a slow atom: one word per lane
        // (host-built unit_codes).  Window octets whose 32 pairs are all class 4 (most
        // of k = 3, 4) take the lean path; the own octet always takes the general one
        // (j > i test).
        const unsigned uw = c.uniform ? 0u : f.unit_codes[32 * U + lane_p];
        const bool slow_u = (uw >> 30) & 1u;
        const unsigned winA = ((uw >> 20) & 0x1fu) | 1u, winB = ((uw >> 25) & 0x1fu) | 1u;
        if (slow_u) {   // the general rounds read the 64-bit codes from shared memory
            unsigned long long code = 0ull;
            if (lane_p < 5) code = f.class_codes[5 * QA + lane_p];
            else if (lane_p >= 8 && lane_p < 13 && QB < nq) code = f.class_codes[5 * QB + lane_p - 8];
            if (lane_p < 5 || (lane_p >= 8 && lane_p < 13)) qcodes[warp][lane_p < 5 ? lane_p : lane_p - 3] = code;
        }
        __syncwarp();
        // packed (quad A, quad B) operands and accumulators of the class-4 rounds
        const float2 oix = make_float2(oiA.x, oiB.x), oiy = make_float2(oiA.y, oiB.y), oiz = make_float2(oiA.z, oiB.z);
        const float2 qKw = make_float2((float)COULOMB_K * oiA.w * c.we[3], (float)COULOMB_K * oiB.w * c.we[3]);
        const float2 Ri = make_float2(riA.x, riB.x), wsi = make_float2(c.wv[3] * riA.y, c.wv[3] * riB.y);
        float2 fx = f2(0.f), fy = f2(0.f), fz = f2(0.f), ee2 = f2(0.f), ev2 = f2(0.f);
        const bool lean = CL_LEAN && !slow_u;
        if (lean) {
            LeanUnit lu;
#if CL_PSTAGE
            // the packed operands pass through the lane's own 8-byte shared slot, so that
            // each arrives as one aligned 64-bit register pair (built in registers, ptxas
            // keeps the halves where the 128-bit loads left them and re-pairs them with two
            // moves per use in every visit: C5 step 0.615 -> 0.608 ms)
            {
                const unsigned ps = smem_u32(&pstage[warp][lane_p]);
                unsigned long long *dst[6] = {&lu.ix, &lu.iy, &lu.iz, &lu.qk, &lu.ri, &lu.se};
                const float lo[6] = {oiA.x, oiA.y, oiA.z, (float)COULOMB_K * oiA.w, riA.x, riA.y};
                const float hi[6] = {oiB.x, oiB.y, oiB.z, (float)COULOMB_K * oiB.w, riB.x, riB.y};
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(ps), "f"(lo[k]), "f"(hi[k]) : "memory");
                    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(*dst[k]) : "r"(ps) : "memory");
                }
            }
#else
            lu.ix = pair_of(oiA.x, oiB.x); lu.iy = pair_of(oiA.y, oiB.y); lu.iz = pair_of(oiA.z, oiB.z);
            lu.qk = pair_of((float)COULOMB_K * oiA.w, (float)COULOMB_K * oiB.w);
            lu.ri = pair_of(riA.x, riB.x);
            lu.se = pair_of(riA.y, riB.y);
#endif
            lu.codes = (uw & 0xfffffu) | ((unsigned)vA << 30) | ((unsigned)vB << 31);
            asm volatile("" : "+r"(lu.codes));   // opaque: the visits test its bits, not re-derive iA < n
            lean_sweep<DCONST, NCAP, EALL>(c, lu, fx, fy, fz, ee2, ev2, ce, cv, U, no, sb, winA | winB, wsb, &xq);
        } else
        for (int ob = U; ob < no; ob += 32) {
            // box pretest of 32 candidate octets at once against the unit's octet box
            const int Oc = ob + lane_p;
            float bd2 = 3.0e38f;
            if (Oc < no) {
                const float4 oc = lds4(sb + L::OCT_C + 16 * Oc), oh = lds4(sb + L::OCT_H + 16 * Oc);
                const float gx = fmaxf(fabsf(cu.x - oc.x) - (hu.x + oh.x), 0.f);
                const float gy = fmaxf(fabsf(cu.y - oc.y) - (hu.y + oh.y), 0.f);
                const float gz = fmaxf(fabsf(cu.z - oc.z) - (hu.z + oh.z), 0.f);
                bd2 = gx * gx + gy * gy + gz * gz;
            }
            unsigned cand = __ballot_sync(FULL, bd2 <= c.pre2);
            const unsigned vmask = __ballot_sync(FULL, bd2 <= c.pre2v);
            // octets in a quad's 64-atom class window (only in the first block) or near
            // a slow atom's tree partner take the general path
            const unsigned genA = slow_u ? ~0u : (ob == U ? winA : 0u);
            const unsigned genB = slow_u ? ~0u : (ob == U ? winB : 0u);
            while (cand) {
                const int t = __ffs(cand) - 1;
                cand &= cand - 1u;
                const int O = ob + t;
                const float4 oc = lds4(sb + L::OCT_C + 16 * O);
                const int j = 8 * O + js;
                const float4 oj = lds4(sb + L::OQ + 16 * j);
                const float2 rj = lds2(sb + L::RS + 8 * j);
                const float sx = cu.x - oc.x, sy = cu.y - oc.y, sz = cu.z - oc.z;   // exact
                const bool vr = (vmask >> t) & 1u;
                float2 gj_x = f2(0.f), gj_y = f2(0.f), gj_z = f2(0.f);
                if (!(((genA | genB) >> t) & 1u)) {
                    // class 4 for both quads: one packed pass over both halves
                    if (!packed_round<DCONST>(c, n, O, iA, iB, vA, vB, lane_p, oix, oiy, oiz, qKw, Ri, wsi, oj, rj, sx,
                                              sy, sz, vr, wnz4, fx, fy, fz, gj_x, gj_y, gj_z, ee2, ev2, ce, cv, exq,
                                              exq_cap, &xq.n))
                        continue;
                } else {
                    // the class window / own octet: both halves' membership first, one vote,
                    // then the math with predicated lanes
                    const Prep pa = prep(f, c, (genA >> t) & 1u, qcodes[warp], n, O, QA, iA, vA, lane_p, oiA, riA, oj,
                                         rj, sx, sy, sz, wnz4, exq, exq_cap, &xq.n);
                    const Prep pb = prep(f, c, (genB >> t) & 1u, qcodes[warp] + 5, n, O, QB, iB, vB, lane_p, oiB, riB,
                                         oj, rj, sx, sy, sz, wnz4, exq, exq_cap, &xq.n);
                    const bool anyA = __any_sync(FULL, pa.fast), anyB = __any_sync(FULL, pb.fast);
                    if (!(anyA | anyB)) continue;
                    if (anyA)
                        pair_math<DCONST>(c, pa, riA, rj, vr, fx.x, fy.x, fz.x, gj_x.x, gj_y.x, gj_z.x, ee2.x, ev2.x, ce,
                                          cv);
                    if (anyB)
                        pair_math<DCONST>(c, pb, riB, rj, vr, fx.y, fy.y, fz.y, gj_x.y, gj_y.y, gj_z.y, ee2.y, ev2.y, ce,
                                          cv);
                }
                float gjx = gj_x.x + gj_x.y, gjy = gj_y.x + gj_y.y, gjz = gj_z.x + gj_z.y;
                // force on j = -(sum over the quad lanes of both halves), once per octet
                gjx += __shfl_xor_sync(FULL, gjx, 1); gjy += __shfl_xor_sync(FULL, gjy, 1);
                gjz += __shfl_xor_sync(FULL, gjz, 1);
                gjx += __shfl_xor_sync(FULL, gjx, 2); gjy += __shfl_xor_sync(FULL, gjy, 2);
                gjz += __shfl_xor_sync(FULL, gjz, 2);
                const float v = ii == 0 ? gjx : (ii == 1 ? gjy : gjz);
                // (padding atoms past n have accumulator words too: NCAP >= 8 no atoms)
                if (ii < 3 && v != 0.f) acc_add<NCAP>(sb, 3 * j + ii, __float2ll_rn(-v * FIXF));
            }
        }
        // i forces: sum over the 8 j-lanes of each i, then into the fixed point
        float fxA = fx.x, fyA = fy.x, fzA = fz.x, fxB = fx.y, fyB = fy.y, fzB = fz.y;
        float ee = ee2.x + ee2.y, ev = ev2.x + ev2.y;
#pragma unroll
        for (int m = 4; m < 32; m <<= 1) {
            fxA += __shfl_xor_sync(FULL, fxA, m); fyA += __shfl_xor_sync(FULL, fyA, m);
            fzA += __shfl_xor_sync(FULL, fzA, m);
            fxB += __shfl_xor_sync(FULL, fxB, m); fyB += __shfl_xor_sync(FULL, fyB, m);
            fzB += __shfl_xor_sync(FULL, fzB, m);
        }
        {
            // lanes js = 0..2 take quad A's x / y / z, js = 4..6 quad B's
            const int q = js & 3;
            const float va = q == 0 ? fxA : (q == 1 ? fyA : fzA), vb = q == 0 ? fxB : (q == 1 ? fyB : fzB);
            const float v = js < 4 ? va : vb;
            const int i = js < 4 ? iA : iB;
            if ((js < 4 ? vA : vB) && q < 3 && v != 0.f) acc_add<NCAP>(sb, 3 * i + q, __float2ll_rn(v * FIXF));
        }
        // the unit's energies (fixed xor tree: deterministic)
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) {
            ee += __shfl_xor_sync(FULL, ee, m);
            ev += __shfl_xor_sync(FULL, ev, m);
        }
        __syncwarp();
        if (lane_p == 0) {
            e_q[2 * U] = (double)ee;
            e_q[2 * U + 1] = (double)ev;
            U = rank + split * atomicAdd(&next_q, 1);
        }
        U = __shfl_sync(FULL, U, 0);
    }
    {
        const int tce = __reduce_add_sync(FULL, ce), tcv = __reduce_add_sync(FULL, cv);
        if (lane_p == 0) { atomicAdd(&cnt_e, (unsigned)tce); atomicAdd(&cnt_v, (unsigned)tcv); }
    }
    __syncthreads();

    // ---- 2b. the queued exact-path pairs: sorted (unique keys: a rank sort), then
    // evaluated in fp64 (forces into the global fixed-point planes), energies summed
    // per thread in sorted order and over the block in a fixed tree: deterministic
    const int m = xq.n;
    double xe = 0.0, xv = 0.0;
    if (m > 0) {
        if (m > exq_cap) {
            if (threadIdx.x == 0 && atomicCAS(&status[b].error, KF_ERR_NONE, KF_ERR_CAPACITY) == KF_ERR_NONE) {
                status[b].err_iter = status[b].iter;
                status[b].overflow = -m;   // negative: the exact-pair queue (not solvation)
            }
        } else {
            unsigned *sorted = exq + exq_cap;
            for (int e = threadIdx.x; e < m; e += CL_THREADS) {
                const unsigned key = exq[e];
                const unsigned k = (key & 0xffffffu) | ((key >> 24) << 30);   // order by (j, i), class last
                int r = 0;
                for (int q = 0; q < m; ++q) {
                    const unsigned o = exq[q];
                    r += ((o & 0xffffffu) | ((o >> 24) << 30)) < k;
                }
                sorted[r] = key;
            }
            __syncthreads();
            const long long plane = 3LL * nbatch * n;
            for (int e = threadIdx.x; e < m; e += CL_THREADS) {
                const unsigned key = sorted[e];
                double se[2] = {0.0, 0.0};
                const int2 k2 = cl_exact_pair(f, pos, (int)(key & 0xfffu), (int)((key >> 12) & 0xfffu),
                                              4 - (int)(key >> 24), planes, plane, (size_t)b * n, status + b, se);
                xe += se[0]; xv += se[1];
                if (k2.x) atomicAdd(&cnt_e, (unsigned)k2.x);
                if (k2.y) atomicAdd(&cnt_v, (unsigned)k2.y);
            }
        }
    }
    xe = warp_sum(xe); xv = warp_sum(xv);
    if (lane == 0) { red_e[warp][0] = xe; red_e[warp][1] = xv; }
    __syncthreads();

    // ---- 3. forces out (+ the exact-path planes if any), energies, counts ----
    namespace cg = cooperative_groups;
    if (split > 1) {
        __threadfence();                 // e_q and the exact-pair planes (global memory)
        cg::this_cluster().sync();       // every CTA of the trajectory is past its sweep
    }
    int mtot = m;
    for (int r = 1; r < split; ++r)
        mtot += cg::this_cluster().map_shared_rank(&xq, (rank + r) % split)->n;
    const bool with_planes = mtot > 0;
    const size_t nb = (size_t)b * n;
    const long long plane = 3LL * nbatch * n;
    const int k0 = (int)((long long)3 * n * rank / split), k1 = (int)((long long)3 * n * (rank + 1) / split);
    for (int k = k0 + threadIdx.x; k < k1; k += CL_THREADS) {
        long long a64 = 0;
        for (int r = 0; r < split; ++r) {   // integer partial sums: the total is order-free
            const unsigned char *smr = split > 1 ? cg::this_cluster().map_shared_rank(sm, r) : sm;
            a64 += ((long long)reinterpret_cast<const int *>(smr + L::ACC_HI)[k] << 40) +
                   ((long long)reinterpret_cast<const unsigned *>(smr + L::ACC_MID)[k] << 20) +
                   (long long)reinterpret_cast<const unsigned *>(smr + L::ACC_LO)[k];
        }
        double v = (double)a64 * FIX_INV;
        if (with_planes) {
            long long *p = planes + 3 * nb + k;
            double *big = reinterpret_cast<double *>(planes + 2 * plane) + 3 * nb + k;
            const long long lo = p[0], hi = p[plane];
            const double bg = *big;
            if (lo || hi || bg != 0.0) {
                v += ((double)hi * FJ_HI + (double)lo * FJ_LO) + bg;
                p[0] = 0; p[plane] = 0; *big = 0.0;
            }
        }
        forces[3 * nb + k] = v;
    }
    if (rank == 0 && warp == 0) {
        double de = 0.0, dv = 0.0;
        for (int q = lane; q < no; q += 32) { de += e_q[2 * q]; dv += e_q[2 * q + 1]; }
        de = warp_sum(de);
        dv = warp_sum(dv);
        long long te = 0, tv = 0;
        for (int r = 0; r < split; ++r) {   // exact pairs: each CTA's warps in order, CTAs in rank order
            const double (*re)[2] = split > 1 ? cg::this_cluster().map_shared_rank(red_e, r) : red_e;
            for (int w2 = 0; w2 < CL_WARPS; ++w2) { de += re[w2][0]; dv += re[w2][1]; }
            te += split > 1 ? *cg::this_cluster().map_shared_rank(&cnt_e, r) : cnt_e;
            tv += split > 1 ? *cg::this_cluster().map_shared_rank(&cnt_v, r) : cnt_v;
        }
        if (lane == 0) {   // doubled: the energy reduction halves (full-list convention)
            e_atom[2 * nb] = 2.0 * de;
            e_atom[2 * nb + 1] = 2.0 * dv;
            pair_count[nb] = 2LL * te + ((2LL * tv) << 32);
        }
    }
    if (split > 1) cg::this_cluster().sync();   // the peers' shared memory outlives every read of it
}

template <bool DCONST, int NCAP, int EALL>
__global__ void __launch_bounds__(CL_WARPS * 32, NCAP <= 1536 ? CL_MINB : 1)
cluster_pair_kernel(const __grid_constant__ kf_field_t f, const __grid_constant__ ClConst c, int n,
                    const double *__restrict__ pos_all, double *__restrict__ forces, double *__restrict__ e_atom,
                    long long *__restrict__ pair_count, kf_status_t *status, long long *__restrict__ planes,
                    unsigned *__restrict__ exq_all, int exq_cap, int nbatch, int split) {
    const int b = blockIdx.x / split, rank = blockIdx.x % split;   // cluster dims (split, 1, 1)
    if (status[b].done) return;
    extern __shared__ __align__(16) unsigned char sm[];
    cluster_pairs_cta<DCONST, NCAP, EALL>(f, c, n, b, pos_all, forces, e_atom, pair_count, status, planes, exq_all,
                                          exq_cap, sm, nbatch, split, rank);
}

// One whole KCM iteration of trajectory b in one CTA (vacuum ensembles on the
// cluster path): forward kinematics (kf_kinematics.cu), the pair phase, then
// wrenches, torques, record, stop tests and the step (kf_torque.cu), with the
// phases separated by block barriers instead of kernel boundaries.  Each CTA
// runs its own chain, so one trajectory's latency-bound FK / torque phases
// overlap the other resident CTA's pair phase, and there is one grid tail per
// iteration instead of three.  The phases reuse one dynamic shared buffer.
template <bool DCONST, int NCAP, int EALL>
__global__ void __launch_bounds__(CL_WARPS * 32, NCAP <= 1536 ? CL_MINB : 1)
fold_iteration_kernel(const __grid_constant__ kf_chain_t ch, const __grid_constant__ kf_field_t f,
                      const __grid_constant__ ClConst c, const __grid_constant__ kf_batch_t w,
                      const __grid_constant__ kf_step_t step, int with_torque, int nbatch) {
    const int b = blockIdx.x;
    if (w.status[b].done) return;
    extern __shared__ __align__(16) unsigned char sm[];
    const int n = ch.n_atoms;
    fk_smem_cta<CL_WARPS * 32>(ch, b, w.theta, w.link_T, w.pos, reinterpret_cast<double *>(sm), 0);
    __syncthreads();
    cluster_pairs_cta<DCONST, NCAP, EALL>(f, c, n, b, w.pos, w.forces, w.e_atom, w.pair_count, w.status, w.pair_fj,
                                          reinterpret_cast<unsigned *>(w.s_lo), 2 * n, sm, nbatch, 1, 0);
    if (!with_torque) return;
    __syncthreads();
    const TorqueArgs ta{w.link_T, w.wrench, w.side_tot, w.bb_suffix, w.tau};
    torque_step_cta<CL_WARPS * 32>(ch, f, ta, w, step, 1, 1, 1, b, reinterpret_cast<double *>(sm));
}

// The field constants KC<2> bakes in (the FieldConfig / WeightTable defaults)
inline bool default_constants(const ClConst &c) {
    return c.mid == 53.f && c.half == 28.f && c.band_l == 1e-3f && c.cutlo == 81.f - 0.95f * 1e-3f &&
           c.tv2 == 25.f && c.close4 == 1.f && c.we[3] == 1.f && c.wv[3] == 1.f && c.uniform == 0;
}

// Small batches: each trajectory is split over a thread-block cluster of S CTAs so
// that the batch still fills two CTAs per SM: S = the largest power of two <= 16
// with B S <= 2 x SMs and at least 8 units per CTA (C1 single: S = 4 27.9 vs S = 8
// 28.9 us; C2 single: S = 16 56.4 vs S = 8 59.4 us); KFB200_CL_SPLIT overrides.
int kf_cluster_split(int B, int n) {
    static int sms = 0, env_split = -1;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const char *e = getenv("KFB200_CL_SPLIT");
        env_split = e ? atoi(e) : 0;
    }
    if (env_split > 0) return env_split;
    int split = 1;
    const int units = (n + 7) / 8;
    while (split < 16 && (long long)B * split * 2 <= 2LL * sms && units >= 16 * split) split *= 2;
    return split;
}

template <int NCAP>
inline int launch_cap(bool dconst, const kf_field_t *f, const ClConst &c, kf_batch_t *w, int n, cudaStream_t s,
                      int plane_b) {
    constexpr size_t smem = ClLayout<NCAP>::TOTAL;
    // EALL: the elec threshold is the pair cut-off (elec >= vdW), so every fp32-path pair has the elec term
    const bool eall = c.te2 >= c.cut2;
    const bool defc = eall && !dconst && default_constants(c);
    auto kern = dconst ? (eall ? cluster_pair_kernel<true, NCAP, 1> : cluster_pair_kernel<true, NCAP, 0>)
                       : (defc ? cluster_pair_kernel<false, NCAP, 2>
                               : eall ? cluster_pair_kernel<false, NCAP, 1> : cluster_pair_kernel<false, NCAP, 0>);
    const int oi = defc ? 4 : 2 * dconst + eall;
    static bool opted[5] = {false, false, false, false, false};
    if (!opted[oi]) {
        KF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "cluster smem");
        // clusters of 16 CTAs (beyond the portable 8) for single short chains
        KF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1), "cluster size");
        opted[oi] = true;
    }
    // exact-pair queue + its sorted copy: the SoA low-word buffer ([B][n][4] u32), which
    // the cluster path does not otherwise use (binning writes it, nothing later reads it)
    const int split = kf_cluster_split(w->B, n);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(w->B * split);
    cfg.blockDim = dim3(CL_WARPS * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = split;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    KF_CUDA(cudaLaunchKernelEx(&cfg, kern, *f, c, n, (const double *)w->pos, w->forces, w->e_atom, w->pair_count,
                               w->status, w->pair_fj, reinterpret_cast<unsigned *>(w->s_lo), 2 * n, plane_b, split),
            "cluster_pair_kernel");
    KF_LAUNCH_CHECK("cluster_pair_kernel");
    return 0;
}

// On error only, cluster path (no cell table was built): smallest (i, j), i < j,
// among pairs at the minimum distance, by a direct sweep (forcefield.py:84-88).
__global__ void cl_clash_report_kernel(kf_field_t f, int B, int n, const double *__restrict__ pos_all,
                                       kf_status_t *status) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (long long)B * n) return;
    const int b = (int)(gid / n), i = (int)(gid % n);
    if (status[b].error != KF_ERR_CLASH) return;
    const double *pos = pos_all + 3 * (size_t)b * n;
    const unsigned long long target = status[b].dmin_bits;
    for (int j = i + 1; j < n; ++j) {
        const double d2 = d2_einsum(xsub(pos[3 * i], pos[3 * j]), xsub(pos[3 * i + 1], pos[3 * j + 1]),
                                    xsub(pos[3 * i + 2], pos[3 * j + 2]));
        if (d2 > f.cut_pair2) continue;
        if ((unsigned long long)__double_as_longlong(sqrt(d2)) == target)
            atomicMin(reinterpret_cast<unsigned long long *>(&status[b].clash_key),
                      ((unsigned long long)i << 32) | (unsigned)j);
    }
}

}  // namespace

int kf_cluster_clash_report_launch(const kf_field_t *f, kf_batch_t *w, int n, cudaStream_t s) {
    const long long total = (long long)w->B * n;
    cl_clash_report_kernel<<<kf_blocks(total, 128), 128, 0, s>>>(*f, w->B, n, w->pos, w->status);
    KF_LAUNCH_CHECK("cl_clash_report_kernel");
    return 0;
}

// The cluster path applies to fp32 pair math on chains that fit one CTA's shared
// memory, at any batch size (small batches split each trajectory over a cluster of
// CTAs).  Measured against the dense lanes: C2 step at B = 128 0.175 vs 0.343 ms,
// B = 32 0.156 vs 0.170; single C2 chain 56.4 vs 60.1 us per iteration (16-CTA
// clusters), C1 28.9 vs 40.1.  KFB200_CLUSTER=0 disables it, KFB200_CLUSTER_MIN_B
// sets a batch threshold (measurements).  kf_bin_launch, kf_pairs_launch and
// kf_torque_launch all consult this, so one launch configuration is consistent.
#ifndef CL_MIN_B
#define CL_MIN_B 1
#endif

int kf_cluster_path(const kf_field_t *f, const kf_batch_t *w, int n) {
    static int env_on = -1, env_min_b = -1;
    static size_t smem_max = 0;
    if (env_on < 0) {
        const char *e = getenv("KFB200_CLUSTER");
        env_on = e ? atoi(e) : 1;
        const char *m = getenv("KFB200_CLUSTER_MIN_B");
        env_min_b = m ? atoi(m) : CL_MIN_B;
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        smem_max = (size_t)v;
    }
    if (!f || !w || !env_on || f->precision || f->flat || !w->pair_fj || n < 1) return 0;
    if (w->B < env_min_b) return 0;
    if (w->api_eval && w->B < 32) return 0;   // single API evaluations: cell lists + dense lanes
    return n <= CL_CAPS[CL_NCAPS - 1] && (size_t)ClLayout<2944>::TOTAL <= smem_max ? 1 : 0;
}

static ClConst cl_const(const kf_field_t *f) {
    ClConst c;
    for (int q = 0; q < 4; ++q) {
        c.we[q] = (float)(f->uniform_weights ? f->uniform_value : f->w_elec[q]);
        c.wv[q] = (float)(f->uniform_weights ? f->uniform_value : f->w_vdw[q]);
    }
    c.band = 1e-3f;
    c.cut2 = (float)f->cut_pair2;
    c.cutlo = c.cut2 - 0.95f * c.band;   // below the band test's reach, whatever its rounding
    c.tv2 = (float)f->thr_vdw2;
    c.te2 = (float)f->thr_elec2;
    c.pre2 = (float)(f->cut_pair2 + 1e-2);
    c.pre2v = (float)(f->thr_vdw2 + 1e-2);
    static float f64_below = -1.f;   // KFB200_PAIR_F64_BELOW (A), as kf_nonbonded.cu
    if (f64_below < 0.f) {
        const char *env = getenv("KFB200_PAIR_F64_BELOW");
        f64_below = env ? (float)atof(env) : 1.0f;
    }
    c.f64_d2 = f64_below * f64_below;
    c.kap_inv = f->dielectric_const ? (float)(1.0 / f->kappa) : 1.0f;
    c.uniform = f->uniform_weights;
    {
        // cut2 = max(elec, vdw)^2 coincides (to an ulp) with the larger per-term
        // threshold, so there are two distinct thresholds; the third one's distance
        // to the nearer of them widens the lean band
        const float t3[3] = {c.cut2, c.tv2, c.te2};
        const float ta = std::min(std::min(t3[0], t3[1]), t3[2]), tb = std::max(std::max(t3[0], t3[1]), t3[2]);
        float dev = 0.f;
        for (float t : t3) dev = std::max(dev, std::min(t - ta, tb - t));
        c.mid = 0.5f * (ta + tb);
        c.half = 0.5f * (tb - ta);
        c.band_l = c.band + dev;
    }
    c.wnz_mask = 0;
    for (int q = 0; q < 4; ++q) {
        c.kwe[q] = (float)COULOMB_K * c.we[q];
        if (c.we[q] != 0.f || c.wv[q] != 0.f) c.wnz_mask |= 1 << q;
    }
    c.close4 = ((c.wnz_mask >> 3) & 1) ? c.f64_d2 : 1e-4f;
    return c;
}

// plane_b: trajectories in the pair_fj planes' stride (w may be a sub-batch view
// of a larger batch, see kf_api.cu batch_view); 0 = w->B
int kf_cluster_pairs_launch(const kf_field_t *f, kf_batch_t *w, int n, cudaStream_t s, int plane_b) {
    const ClConst c = cl_const(f);
    const bool dc = f->dielectric_const != 0;
    if (plane_b <= 0) plane_b = w->B;
    if (n <= 512) return launch_cap<512>(dc, f, c, w, n, s, plane_b);
    if (n <= 1024) return launch_cap<1024>(dc, f, c, w, n, s, plane_b);
    if (n <= 1536) return launch_cap<1536>(dc, f, c, w, n, s, plane_b);
    if (n <= 2048) return launch_cap<2048>(dc, f, c, w, n, s, plane_b);
    return launch_cap<2944>(dc, f, c, w, n, s, plane_b);
}

template <int NCAP>
static int launch_fused(const kf_chain_t *ch, const kf_field_t *f, kf_batch_t *w, const kf_step_t *st,
                        cudaStream_t s, int with_torque, int plane_b) {
    const ClConst c = cl_const(f);
    const bool dc = f->dielectric_const != 0;
    size_t smem = ClLayout<NCAP>::TOTAL;
    smem = std::max(smem, fk_smem_bytes(*ch));
    smem = std::max(smem, (size_t)ch->n_links * 6 * sizeof(double));
    const bool eall = c.te2 >= c.cut2;
    const bool defc = eall && !dc && default_constants(c);
    auto kern = dc ? (eall ? fold_iteration_kernel<true, NCAP, 1> : fold_iteration_kernel<true, NCAP, 0>)
                   : (defc ? fold_iteration_kernel<false, NCAP, 2>
                           : eall ? fold_iteration_kernel<false, NCAP, 1> : fold_iteration_kernel<false, NCAP, 0>);
    KF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "fused smem");
    kern<<<w->B, CL_WARPS * 32, smem, s>>>(*ch, *f, c, *w, *st, with_torque, plane_b > 0 ? plane_b : w->B);
    KF_LAUNCH_CHECK("fold_iteration_kernel");
    return with_torque ? 0 : 2;
}

// The fused iteration (KFB200_FUSED=1) applies to vacuum ensembles on the cluster
// path whose chain fits (single-CTA FK and torque phases, wrenches in shared
// memory).  Off by default: measured on C5, 1.21 ms per iteration fused vs 1.15
// ms as three kernels.  Both resident CTAs of an SM tend to sit in their
// latency-bound FK / torque phases together, and those phases run at 2 CTAs per
// SM instead of the standalone kernels' 4.
// KFB200_FUSED=2: FK and the pair phase fused (torques a separate kernel; returns 2).
int kf_fused_iteration(const kf_chain_t *ch, const kf_field_t *f, kf_batch_t *w, const kf_step_t *st, cudaStream_t s,
                       int plane_b) {
    static int env_on = -1;
    if (env_on < 0) {
        const char *e = getenv("KFB200_FUSED");
        env_on = e ? atoi(e) : 0;
    }
    const int n = ch->n_atoms;
    if (!env_on || f->solvation || !st || !kf_cluster_path(f, w, n) || kf_cluster_split(w->B, n) != 1) return -1;
    if (fk_smem_bytes(*ch) > 200 * 1024 || (size_t)ch->n_links * 48 > 200 * 1024) return -1;
    const int wt = env_on == 2 ? 0 : 1;
    if (n <= 512) return launch_fused<512>(ch, f, w, st, s, wt, plane_b);
    if (n <= 1024) return launch_fused<1024>(ch, f, w, st, s, wt, plane_b);
    if (n <= 1536) return launch_fused<1536>(ch, f, w, st, s, wt, plane_b);
    if (n <= 2048) return launch_fused<2048>(ch, f, w, st, s, wt, plane_b);
    return launch_fused<2944>(ch, f, w, st, s, wt, plane_b);
}
