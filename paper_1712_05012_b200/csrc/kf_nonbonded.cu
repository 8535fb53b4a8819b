// Nonbonded elec + vdW pair kernel (K3) with the cut-off filter (K2), the
// 1-2/1-3/1-4 classifier and the steric-clash guard fused in.
//
// Reference: Field.evaluate's force phase (/root/reference/pkg/src/kinefold/
// kcm.py:110-127) = extract_pairs (forcefield.py:81-89 -> spatial.py:233-241),
// TreeWeights.weights_for (topology.py:153-195), elec/vdw_pair_quantities
// (forcefield.py:98-113) and the bincount scatter (forcefield.py:162-172).
//
// Work items are (occupied 9 A cell, 32-atom i-chunk of it) over all
// trajectories, taken from a dynamic counter: one warp per item (ensembles) or
// one CTA per item whose warps share the j-tiles (SPLIT: small batches).
// Per item the warp probes the 27 neighbour cells at once (lane = stencil
// cell), keeps those whose bounding box some i of the chunk reaches, and
// concatenates their atoms into one j-stream cut into full 32-atom tiles
// (positions shifted into the i cell's frame while staging).  Per tile:
//   1. prefilter: lane = j, loop over the chunk's i (broadcast), fp32 d^2
//      against cut^2 + 1e-2 A^2; a ballot per i gives owner i's 32-bit row;
//   2. compacted pairs: the set bits of all rows are dealt out one pair per
//      lane, owner-major (warp scan + bit walk), so every lane does useful
//      pair work; each pair gets its difference vector from the hi/lo fp32
//      offset pairs (fp64-accurate), decides membership exactly as the
//      reference (d2 = (dx*dx + dz*dz) + dy*dy in fp64 vs max(elec, vdw)^2,
//      and sqrt(d2) <= cut per term) -- recomputed from the fp64 positions
//      only in a 1e-3 A^2 band around each threshold -- and evaluates energy
//      and force in fp32; pairs under 1 A take the reference's fp64 formulas.
//   The per-pair results are summed per owner lane in pair order, i.e. in a
//   fixed order, into fp64 accumulators.
// Both directions of each unordered pair are evaluated by their owners
// ("full list"): no atomics on forces, run-to-run bitwise deterministic.
#include <cstdlib>
#include <type_traits>

#include "kf_common.cuh"

namespace {

constexpr double COULOMB_K = 332.06;
constexpr double MIN_DISTANCE = 1e-6;
// two-level fixed point of the half-list kernel's j-side forces: hi in units of
// 2^12, lo (the exact remainder, |r| <= 2^11) in units of 2^-28
constexpr double FJ_HI = 4096.0, FJ_HI_INV = 1.0 / 4096.0;
constexpr double FJ_LO = 1.0 / 268435456.0, FJ_LO_INV = 268435456.0;
// beyond this magnitude a contribution would overflow the hi plane's int64 once a
// few are summed (|hi| <= 2^60 each): it goes to the fp64 plane instead (pairs
// closer than ~0.05 A only)
constexpr double FJ_SAT = 4722366482869645213696.0;   // 2^72
constexpr int PAIR_WARPS = 4;        // warps per CTA, warp-per-cell variant
constexpr int SPLIT_WARPS = 4;       // warps per CTA (one cell), split variant
constexpr unsigned FULL = 0xffffffffu;


// Adds v to one component of the half-list kernel's j-side accumulator:
// planes = [lo int64 | hi int64 | big fp64], each [B][n][3], plane = 3 B n.
// Integer atomics are order-free, so the sum is schedule-independent; only
// |v| >= 2^72 (never a fast-path pair) takes the fp64 atomic.
KF_DEV void fj_add(long long *planes, long long plane, size_t idx, double v) {
    if (v == 0.0) return;
    if (!(fabs(v) < FJ_SAT)) {
        atomicAdd(reinterpret_cast<double *>(planes + 2 * plane + idx), v);
        return;
    }
    const long long hi_u = __double2ll_rn(v * FJ_HI_INV);     // units of 2^12
    const double rem = v - (double)hi_u * FJ_HI;               // exact, |rem| <= 2^11
    const long long lo_u = __double2ll_rn(rem * FJ_LO_INV);    // units of 2^-28
    if (lo_u) atomicAdd(reinterpret_cast<unsigned long long *>(planes + idx), (unsigned long long)lo_u);
    if (hi_u) atomicAdd(reinterpret_cast<unsigned long long *>(planes + plane + idx), (unsigned long long)hi_u);
}

struct Tile {
    float4 hi[32];
    float4 lo[32];
    float4 par[32];
    int4 aux[32];
};

#ifndef RES_BATCH_N
#define RES_BATCH_N 128
#endif
constexpr int RES_BATCH = RES_BATCH_N;

template <typename T>
struct WarpSmem {
    Tile J;
    T res[RES_BATCH][3];       // per-pair forces of the current batch of the tile's list
    unsigned short list[1024]; // candidate (owner << 5 | t) pairs of the tile, owner-major
};


// fp32 constants of the fast path, passed by value (kernel parameter space:
// constant-bank operands, no registers).
struct PairConst {
    float we[4], wv[4];          // elec / vdW weight by class 1..4
    float pre2, cut2, tv2, te2;  // prefilter and cut-offs (A^2)
    float kap_inv, cell;
    float f64_d2;                // pairs closer than this (A^2) take the fp64 formulas
    int dconst, uniform;
    int te_is_cut;               // elec threshold within 1e-6 A^2 of the pair cut-off
};

__device__ __noinline__ int slow_class(const int32_t *tp, const int32_t *tgp, const int32_t *tgg,
                                       const int32_t *tres, const uint8_t *tchain, int i, int j) {
    if (!tchain[i] || !tchain[j] || abs(tres[i] - tres[j]) > 1) return 4;
    const int pi = tp[i], gpi = tgp[i], ggi = tgg[i], pj = tp[j], gpj = tgp[j], ggj = tgg[j];
    if (pi == j || pj == i) return 1;
    if (gpi == j || gpj == i || (pi >= 0 && pi == pj)) return 2;
    if (ggi == j || ggj == i || (gpi >= 0 && gpi == pj) || (gpj >= 0 && gpj == pi)) return 3;
    return 4;
}

template <typename T>
__device__ __noinline__ void slow_pair(bool f64, const kf_field_t *A, const double4 *pi_, const double4 *pj_, int i,
                                       int j, int cls, T *out, int *pce, int *pcv, kf_status_t *st) {
    const double4 p_i = *pi_, p_j = *pj_;
    const double dx = xsub(p_i.x, p_j.x), dy = xsub(p_i.y, p_j.y), dz = xsub(p_i.z, p_j.z);
    const double d2 = d2_einsum(dx, dy, dz);
    if (d2 > A->cut_pair2) return;
    const bool ke = d2 <= A->thr_elec2, kv = d2 <= A->thr_vdw2;
    *pce = ke; *pcv = kv;
    const double we = A->uniform_weights ? A->uniform_value : A->w_elec[cls - 1];
    const double wv = A->uniform_weights ? A->uniform_value : A->w_vdw[cls - 1];
    if (d2 < 1e-11) {
        const double d = sqrt(d2);
        if (d < MIN_DISTANCE) {
            atomicMin(&st->dmin_bits, (unsigned long long)__double_as_longlong(d));
            if (atomicCAS(&st->error, KF_ERR_NONE, KF_ERR_CLASH) == KF_ERR_NONE) st->err_iter = st->iter;
            return;
        }
    }
    const double d = sqrt(d2);
    const double inv_d = 1.0 / d;
    double mag = 0.0, ee = 0.0, ev = 0.0;
    if (ke) {
        const double num = COULOMB_K * we * A->q[i] * A->q[j];
        ee = A->dielectric_const ? num * inv_d / A->kappa : num * inv_d * inv_d;   // num / (kappa d)
        mag += ee * inv_d;                                              // num / (kappa d^2)
    }
    if (kv) {
        const double eps = sqrt(A->eps[i] * A->eps[j]);
        const double r = (A->R[i] + A->R[j]) * inv_d;
        const double r2 = r * r, r6 = r2 * r2 * r2;
        ev = wv * eps * (r6 * r6 - 2.0 * r6);
        mag += 12.0 * wv * eps * (r6 * r6 - r6) * inv_d;
    }
    const double g = mag * inv_d;
    out[0] = (T)(g * dx); out[1] = (T)(g * dy); out[2] = (T)(g * dz);
    out[3] = (T)ee; out[4] = (T)ev;
    (void)f64;
}

// One ordered pair (owner i, partner j) of the fast path: difference vector
// from the hi/lo fp32 offsets, the reference's membership tests, the static
// class window, and fp32 energy/force -- with the exact fp64 recomputation in
// the 1e-3 A^2 threshold bands and below f64_d2 (always, in fp64 mode).
// out = force on i (x, y, z), elec and vdW energy.  Shared by both kernels.
// Returns true when the exact fp64 path ran: its results are then in sd[5]
// (fp64, never rounded to T: clash-range forces overflow fp32) and out[] is 0.
template <bool F64, typename T>
KF_DEV bool pair_eval(const kf_field_t &f, const PairConst &pc, float4 hi, float4 li, float4 qi, int4 ai, int4 cm,
                      float4 hj, float4 lj, float4 qj, int4 aj, const double4 *pos_i, const double4 *pos_j,
                      kf_status_t *st, T out[5], int &pce, int &pcv, double sd[5]) {
    const float cut2f = pc.cut2, tvf = pc.tv2, tef = pc.te2;
    const float band = 1e-3f;
    const int i = ai.x, j = aj.x;
    const float dxf = (hi.x - hj.x) + (li.x - lj.x);
    const float dyf = (hi.y - hj.y) + (li.y - lj.y);
    const float dzf = (hi.z - hj.z) + (li.z - lj.z);
    const float d2f = dxf * dxf + dyf * dyf + dzf * dzf;
    if (i == j || d2f > cut2f + band) return false;
    // static class window: 2-bit codes for j - i in [-32, 32)
    int cls = 4;
    if (!pc.uniform) {
        const int off = j - i + 32;
        if ((unsigned)off < 64u) {
            const unsigned wd = off < 32 ? (off < 16 ? cm.x : cm.y) : (off < 48 ? cm.z : cm.w);
            cls = 4 - (int)((wd >> (2 * (off & 15))) & 3u);
        } else if (ai.w != 0 && aj.z != 0 && abs(ai.y - aj.y) <= 1) {
            cls = slow_class(f.tparent, f.tgp, f.tggp, f.tres, f.tchain, i, j);
        }
    }
    const float we = pc.we[cls - 1], wv = pc.wv[cls - 1];   // constant-bank loads, indexed
    // exact recomputation near a threshold: |d2 - t| <= band for t in {cut, te, tv}
    // (te == cut to ~1e-14 for the default cut-offs: pc.te_is_cut folds the test)
    // non-short-circuit: predicated compares instead of a branch per threshold
    const bool exact = F64 || ((fabsf(d2f - cut2f) <= band) | (fabsf(d2f - tvf) <= band) |
                               (!pc.te_is_cut & (fabsf(d2f - tef) <= band)) | (d2f < pc.f64_d2));
    if (exact) {
        // the outlined path writes through pointers: give it its own stack
        // temporaries so out / pce / pcv stay in registers on the fast path
        double so[5] = {0, 0, 0, 0, 0};
        int sce = 0, scv = 0;
        slow_pair<double>(F64, &f, pos_i, pos_j, i, j, cls, so, &sce, &scv, st);
        sd[0] = so[0]; sd[1] = so[1]; sd[2] = so[2]; sd[3] = so[3]; sd[4] = so[4];
        pce = sce; pcv = scv;
        return true;
    }
    // (here d2f < cut2f - band: nearer the cut-off went exact, beyond it returned above)
    const bool ke = d2f <= tef, kv = d2f <= tvf;
    pce = ke; pcv = kv;
    // MUFU.RSQ without the subnormal fix-up rsqrtf carries: d2f >= f64_d2 > 0
    // here (closer pairs took the exact path), so the result is the same
    float inv_r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(inv_r) : "f"(d2f));
    const float inv_r2 = inv_r * inv_r;
    // both terms evaluated and selected (no divergent branches; same values)
    // kappa = d: E = K w qi qj / d^2; constant: E = K w qi qj / (kappa d);
    // |F| / d = E / d^2 in both cases
    const float qq = (float)COULOMB_K * qi.x * qj.x * we;
    const float e = pc.dconst ? qq * pc.kap_inv * inv_r : qq * inv_r2;
    const float weps = wv * qi.z * qj.z;
    const float D = qi.y + qj.y;
    const float sr = D * D * inv_r2;
    const float s3 = sr * sr * sr;
    const float s6 = s3 * s3;
    out[3] = ke ? e : 0.f;
    out[4] = kv ? weps * (s6 - 2.f * s3) : 0.f;
    // g = e / d^2, then + 12 w eps (s6 - s3) / d^2 as one FFMA (the rounding of the
    // branchy form: fp32 trajectories are chaotic, keep their rounding stable)
    float g = ke ? e * inv_r2 : 0.f;
    g = kv ? __fmaf_rn(12.f * weps * (s6 - s3), inv_r2, g) : g;
    out[0] = g * dxf; out[1] = g * dyf; out[2] = g * dzf;
    return false;
}

#ifndef PAIR_MINB_W
#define PAIR_MINB_W 5   // resident CTAs per SM asked of ptxas, warp-per-chunk variant
#endif
// F64 = false: fp32 pair math (the north-star configuration); true: fp64
// pair math and fp64 per-tile sums (strict trajectory parity mode).
// SPLIT = true: one CTA per cell, its 4 warps split the 27 neighbour cells
// (short per-cell latency: single trajectories); false: one warp per cell
// (throughput: ensembles).
template <bool F64, bool SPLIT>
__global__ void __launch_bounds__((SPLIT ? SPLIT_WARPS : PAIR_WARPS) * 32, SPLIT ? 1 : PAIR_MINB_W)
pair_kernel(const __grid_constant__ kf_field_t f, const __grid_constant__ PairConst pc, int B, int n, int chunk, const unsigned long long *__restrict__ keys,
            const int32_t *__restrict__ cnt, const int32_t *__restrict__ start, const int32_t *__restrict__ occ,
            const int32_t *__restrict__ occ_count, const int32_t *__restrict__ chunk_pre,
            const int32_t *__restrict__ item_cell,
            const int32_t *__restrict__ chunk_offset, const float4 *__restrict__ s_hi,
            const float4 *__restrict__ s_lo, const double4 *__restrict__ s_pos, const float4 *__restrict__ s_par,
            const int4 *__restrict__ s_aux, const int4 *__restrict__ s_tree, const float4 *__restrict__ cell_box,
            int32_t *__restrict__ work, double *__restrict__ forces, double *__restrict__ e_atom,
            long long *__restrict__ pair_count, kf_status_t *status) {
    using T = typename std::conditional<F64, double, float>::type;
    constexpr int NW = SPLIT ? SPLIT_WARPS : PAIR_WARPS;
    constexpr int NI = SPLIT ? 1 : NW;
    __shared__ Tile Itile[NI];               // the i-chunk (shared by the CTA's warps if SPLIT)
    __shared__ int4 itree_s[NI][32];
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    WarpSmem<T> *smem = reinterpret_cast<WarpSmem<T> *>(dyn_smem);   // [NW]
    __shared__ double part[SPLIT ? NW : 1][3][32];
    __shared__ double epart[NW][2];
    __shared__ long long cpart[NW];
    __shared__ int item_s[NW];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem<T> &S = smem[warp];
    Tile &I = Itile[SPLIT ? 0 : warp];
    int4 *itree = itree_s[SPLIT ? 0 : warp];
    const uint32_t H = 1u << f.hash_bits;
    const int total = chunk_offset[B];
    const float cellf = pc.cell, pre2 = pc.pre2, cut2f = pc.cut2, tvf = pc.tv2, tef = pc.te2;
    const float band = 1e-3f;

    for (;;) {
        int item;
        if (SPLIT) {
            __syncthreads();
            if (threadIdx.x == 0) item_s[0] = atomicAdd(work, 1);
            __syncthreads();
            item = item_s[0];
        } else {
            item = 0;
            if (lane == 0) item = atomicAdd(work, 1);
            item = __shfl_sync(FULL, item, 0);
        }
        if (item >= total) break;
        // item -> (trajectory, occupied cell, 32-atom i-chunk of that cell)
        const int b = item_owner(chunk_offset, B, item);
        const size_t hb = (size_t)b * H, nb = (size_t)b * n;
        const int local = item - chunk_offset[b];
        const int klo = item_cell[hb + local];        // the item's cell (list position)
        const int slot = occ[hb + klo];
        const int ic = (local - chunk_pre[hb + klo]) * chunk;
        int cx, cy, cz;
        unpack_cell((long long)keys[hb + slot], cx, cy, cz);
        const int s0 = start[hb + slot], c = cnt[hb + slot];
        double ee = 0.0, ev = 0.0;   // chunk totals (per computing lane)
        int ce = 0, cv = 0;          // elec / vdW cut-off partners (per computing lane)
        {
            const int ci_n = min(chunk, c - ic);
            const bool valid = lane < ci_n;
            if ((!SPLIT || warp == 0) && valid) {
                const size_t ki = nb + s0 + ic + lane;
                I.hi[lane] = s_hi[ki];
                I.lo[lane] = s_lo[ki];
                I.par[lane] = s_par[ki];
                I.aux[lane] = s_aux[ki];
                itree[lane] = s_tree[ki];
            }
            if (SPLIT) __syncthreads(); else __syncwarp();
            double ax = 0.0, ay = 0.0, az = 0.0;   // owner lane: fp64 force sums over the chunk's tiles

            // probe all neighbour cells at once (lane s <-> stencil cell s) and keep
            // the cells whose bounding box some i of the chunk can reach
            // (warp-uniform loop over the chunk's atoms: no lane-dependent trip
            // counts ahead of the warp collectives below)
            int p_j0 = 0, p_jc = 0, p_js = -1;
            float p_sx = 0.f, p_sy = 0.f, p_sz = 0.f;
            float4 blo = make_float4(1e30f, 1e30f, 1e30f, 0.f), bhi = make_float4(-1e30f, -1e30f, -1e30f, 0.f);
            if (lane < f.n_stencil) {
                const int ox = f.stencil[3 * lane], oy = f.stencil[3 * lane + 1], oz = f.stencil[3 * lane + 2];
                p_js = cell_probe(keys + hb, H, cx + ox, cy + oy, cz + oz);
                if (p_js >= 0) {
                    p_sx = (float)ox * cellf; p_sy = (float)oy * cellf; p_sz = (float)oz * cellf;
                    blo = cell_box[2 * (hb + p_js)]; bhi = cell_box[2 * (hb + p_js) + 1];
                }
            }
            __syncwarp();
            bool keep = false;
            for (int q = 0; q < ci_n; ++q) {
                const float4 r = I.hi[q];   // i in the neighbour cell's frame
                const float px = r.x - p_sx, py = r.y - p_sy, pz = r.z - p_sz;
                const float gx = fmaxf(fmaxf(blo.x - px, px - bhi.x), 0.f);
                const float gy = fmaxf(fmaxf(blo.y - py, py - bhi.y), 0.f);
                const float gz = fmaxf(fmaxf(blo.z - pz, pz - bhi.z), 0.f);
                keep |= gx * gx + gy * gy + gz * gz <= pre2;
            }
            if (keep) { p_j0 = start[hb + p_js]; p_jc = cnt[hb + p_js]; }
            // the kept cells' atoms form one j-stream (stencil order), cut into
            // full 32-atom tiles; tiles are dealt to the CTA's warps round-robin
            int p_end = p_jc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(FULL, p_end, o);
                if (lane >= o) p_end += v;
            }
            const int n_stream = __shfl_sync(FULL, p_end, 31);
            for (int jb = SPLIT ? 32 * warp : 0; jb < n_stream; jb += SPLIT ? 32 * NW : 32) {
                const int nt = min(32, n_stream - jb);
                {
                    // lane -> stream element jb + lane -> (stencil cell, atom): first cell whose end exceeds it
                    const int e = jb + lane;
                    int cs = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        const int end = __shfl_sync(FULL, p_end, cs + step - 1);
                        if (end <= e) cs += step;
                    }
                    const int cend = __shfl_sync(FULL, p_end, cs), cj0 = __shfl_sync(FULL, p_j0, cs),
                              ccnt = __shfl_sync(FULL, p_jc, cs);
                    const float ssx = __shfl_sync(FULL, p_sx, cs), ssy = __shfl_sync(FULL, p_sy, cs),
                                ssz = __shfl_sync(FULL, p_sz, cs);
                    __syncwarp();
                    if (lane < nt) {
                        const int kk = cj0 + (e - (cend - ccnt));
                        const size_t kj = nb + kk;
                        const float4 h = s_hi[kj];
                        int4 aux = s_aux[kj];
                        aux.w = kk;                     // sorted index (fp64 slow path)
                        S.J.hi[lane] = make_float4(h.x + ssx, h.y + ssy, h.z + ssz, 0.f);   // i's cell frame
                        S.J.lo[lane] = s_lo[kj];
                        S.J.par[lane] = s_par[kj];
                        S.J.aux[lane] = aux;
                    }
                    __syncwarp();
                }
                // ---- stage 1: fp32 prefilter, j per lane, i broadcast; lane o keeps owner o's row
                unsigned mask = 0u;
                {
                    const float4 rj = S.J.hi[lane < nt ? lane : 0];
                    for (int q = 0; q < ci_n; ++q) {
                        const float4 r = I.hi[q];
                        const float dx = r.x - rj.x, dy = r.y - rj.y, dz = r.z - rj.z;
                        const unsigned row = __ballot_sync(FULL, lane < nt && dx * dx + dy * dy + dz * dz <= pre2);
                        if (lane == q) mask = row;
                    }
                }
                    // ---- stage 2: the tile's candidate pairs, owner-major, one per lane
                    const int own = __popc(mask);
                    int incl = own;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int v = __shfl_up_sync(FULL, incl, o);
                        if (lane >= o) incl += v;
                    }
                    const int tot = __shfl_sync(FULL, incl, 31);
                    {
                        unsigned m = mask;
                        int wpos = incl - own;
                        while (m) {
                            const int t = __ffs(m) - 1;
                            m &= m - 1u;
                            S.list[wpos++] = (unsigned short)((lane << 5) | t);
                        }
                    }
                    __syncwarp();
                    T fe = 0, fv = 0;
                    T fx = 0, fy = 0, fz = 0;   // owner sums of this tile
                    const int excl = incl - own;
                    for (int base = 0; base < tot; base += RES_BATCH) {
                      const int nbat = min(RES_BATCH, tot - base);
                      for (int k0 = 0; k0 < nbat; k0 += 32) {
                        const int k = base + k0 + lane;
                        const bool act = k0 + lane < nbat;
                        const int e = act ? (int)S.list[k] : 0;
                        const int o = act ? e >> 5 : 32 + lane;   // inactive lanes: own segments
                        T out[5] = {0, 0, 0, 0, 0};
                        int pce = 0, pcv = 0;
                        if (act) {
                            const int t = e & 31;
                            const int4 ai = I.aux[o], aj = S.J.aux[t];
                            const float4 hi = I.hi[o], li = I.lo[o], hj = S.J.hi[t], lj = S.J.lo[t];
                            double sd[5];
                            if (pair_eval<F64, T>(f, pc, hi, li, I.par[o], ai, itree[o], hj, lj, S.J.par[t], aj,
                                                  s_pos + nb + s0 + ic + o, s_pos + nb + aj.w, status + b, out, pce,
                                                  pcv, sd))
                                for (int q = 0; q < 5; ++q) out[q] = (T)sd[q];   // fp64 mode: T = double
                        }
                        // energies and counts only enter per-chunk totals: the computing lane keeps them
                        fe += out[3]; fv += out[4];
                        ce += pce; cv += pcv;
                        if (act) { S.res[k0 + lane][0] = out[0]; S.res[k0 + lane][1] = out[1]; S.res[k0 + lane][2] = out[2]; }
                      }
                      __syncwarp();
                      // each owner sums its contiguous range of the list in order (deterministic)
                      const int lo_k = max(excl - base, 0), hi_k = min(incl - base, nbat);
                      for (int q = lo_k; q < hi_k; ++q) { fx += S.res[q][0]; fy += S.res[q][1]; fz += S.res[q][2]; }
                      __syncwarp();
                    }
                    ax += (double)fx; ay += (double)fy; az += (double)fz;
                    ee += (double)fe; ev += (double)fv;
                }
            if (SPLIT) {
                // combine the warps' partial forces in warp order (deterministic)
                part[SPLIT ? warp : 0][0][lane] = ax;
                part[SPLIT ? warp : 0][1][lane] = ay;
                part[SPLIT ? warp : 0][2][lane] = az;
                __syncthreads();
                if (warp == 0 && valid) {
                    double fx = 0.0, fy = 0.0, fz = 0.0;
#pragma unroll
                    for (int w = 0; w < (SPLIT ? NW : 1); ++w) {
                        fx += part[w][0][lane]; fy += part[w][1][lane]; fz += part[w][2][lane];
                    }
                    const size_t o = nb + I.aux[lane].x;
                    forces[3 * o] = fx; forces[3 * o + 1] = fy; forces[3 * o + 2] = fz;
                    e_atom[2 * o] = 0.0; e_atom[2 * o + 1] = 0.0;
                    pair_count[o] = 0;
                }
                __syncthreads();
            } else if (valid) {
                const size_t o = nb + I.aux[lane].x;
                forces[3 * o] = ax; forces[3 * o + 1] = ay; forces[3 * o + 2] = az;
                e_atom[2 * o] = 0.0; e_atom[2 * o + 1] = 0.0;
                pair_count[o] = 0;
            }
        }
        long long pcount = (long long)ce + ((long long)cv << 32);
        // chunk totals: fixed xor tree per warp, then warps in order, stored at the
        // chunk's first atom (chunks are a function of the positions: deterministic)
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            ee += __shfl_xor_sync(FULL, ee, d);
            ev += __shfl_xor_sync(FULL, ev, d);
            pcount += __shfl_xor_sync(FULL, pcount, d);
        }
        if (SPLIT) {
            if (lane == 0) { epart[warp][0] = ee; epart[warp][1] = ev; cpart[warp] = pcount; }
            __syncthreads();
            if (threadIdx.x == 0) {
                double te = 0.0, tv = 0.0;
                long long tc = 0;
                for (int w = 0; w < NW; ++w) { te += epart[w][0]; tv += epart[w][1]; tc += cpart[w]; }
                const size_t o = nb + s_aux[nb + s0 + ic].x;
                e_atom[2 * o] = te; e_atom[2 * o + 1] = tv;
                pair_count[o] = tc;
            }
        } else {
            __syncwarp();
            if (lane == 0) {
                const size_t o = nb + s_aux[nb + s0 + ic].x;
                e_atom[2 * o] = ee; e_atom[2 * o + 1] = ev;
                pair_count[o] = pcount;
            }
        }
    }
}

// ---- dense variant --------------------------------------------------------
//
// Same work items, probes and j-stream as pair_kernel, but no compaction: lane
// = owner i (its data in registers), the j-tile is broadcast from shared
// memory.  Chunks of <= 16 (<= 8) atoms are duplicated across 2 (4) lane
// groups that take alternating j, so more lanes work; the groups' fp64 sums are
// combined by a fixed xor tree at the end of the item.  Each lane sums its
// own pairs in j order: deterministic, no per-pair shared-memory traffic.
template <bool F64, bool SPLIT, bool HALF>
__global__ void __launch_bounds__((SPLIT ? SPLIT_WARPS : PAIR_WARPS) * 32, SPLIT ? 1 : PAIR_MINB_W)
pair_dense_kernel(const __grid_constant__ kf_field_t f, const __grid_constant__ PairConst pc, int B, int n, int chunk,
                  const unsigned long long *__restrict__ keys, const int32_t *__restrict__ cnt,
                  const int32_t *__restrict__ start, const int32_t *__restrict__ occ,
                  const int32_t *__restrict__ occ_count, const int32_t *__restrict__ chunk_pre,
            const int32_t *__restrict__ item_cell,
                  const int32_t *__restrict__ chunk_offset, const float4 *__restrict__ s_hi,
                  const float4 *__restrict__ s_lo, const double4 *__restrict__ s_pos,
                  const float4 *__restrict__ s_par, const int4 *__restrict__ s_aux, const int4 *__restrict__ s_tree,
                  const float4 *__restrict__ cell_box, int32_t *__restrict__ work, double *__restrict__ forces,
                  double *__restrict__ e_atom, long long *__restrict__ pair_count, kf_status_t *status,
                  long long *__restrict__ fj_fixed) {
    kf_pdl_wait();      // after the predecessor (programmatic launch: single trajectories)
    kf_pdl_trigger();
    const long long fj_plane = 3LL * B * n;
    using T = typename std::conditional<F64, double, float>::type;
    constexpr int NW = SPLIT ? SPLIT_WARPS : PAIR_WARPS;
    __shared__ Tile Jt[NW];
    // HALF: per lane, its contribution to each j of the tile ([x|y|z][t][owner slot],
    // chunks of <= 16 atoms); summed per j in owner order at the end of the tile
    __shared__ __align__(16) float Jc_s[HALF ? NW : 1][3][32][16];
    __shared__ float4 ihi_s[SPLIT ? 1 : NW][32];   // the chunk's hi offsets (probe / box test)
    __shared__ double part[SPLIT ? NW : 1][3][32];
    __shared__ double epart[NW][2];
    __shared__ long long cpart[NW];
    __shared__ int item_s[1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Tile &J = Jt[warp];
    float4 *ihi = ihi_s[SPLIT ? 0 : warp];
    const uint32_t H = 1u << f.hash_bits;
    const int total = chunk_offset[B];
    const float cellf = pc.cell, pre2 = pc.pre2;

    for (;;) {
        int item;
        if (SPLIT) {
            __syncthreads();
            if (threadIdx.x == 0) item_s[0] = atomicAdd(work, 1);
            __syncthreads();
            item = item_s[0];
        } else {
            item = 0;
            if (lane == 0) item = atomicAdd(work, 1);
            item = __shfl_sync(FULL, item, 0);
        }
        if (item >= total) break;
        // item -> (trajectory, occupied cell, 32-atom i-chunk of that cell)
        const int b = item_owner(chunk_offset, B, item);
        const size_t hb = (size_t)b * H, nb = (size_t)b * n;
        const int local = item - chunk_offset[b];
        const int klo = item_cell[hb + local];        // the item's cell (list position)
        const int slot = occ[hb + klo];
        const int ic = (local - chunk_pre[hb + klo]) * chunk;
        int cx, cy, cz;
        unpack_cell((long long)keys[hb + slot], cx, cy, cz);
        const int s0 = start[hb + slot], c = cnt[hb + slot];
        const int ci_n = min(chunk, c - ic);
        // lane -> (owner slot, j phase): chunks of <= 16 / 8 / 4 / 2 atoms use 2 / 4 / 8 / 16 phases
        const int nph = ci_n > 16 ? 1 : ci_n > 8 ? 2 : ci_n > 4 ? 4 : ci_n > 2 ? 8 : 16;
        const int wi = 32 / nph, oi = lane % wi, ph = lane / wi;
        const bool own = oi < ci_n;
        const size_t ki = nb + s0 + ic + (own ? oi : 0);
        const float4 hi = s_hi[ki], li = s_lo[ki], qi = s_par[ki];
        const int4 ai = s_aux[ki], cm = s_tree[ki];
        if ((!SPLIT || warp == 0) && lane < ci_n) ihi[lane] = s_hi[nb + s0 + ic + lane];
        if (SPLIT) __syncthreads(); else __syncwarp();

        // probe the 27 neighbour cells (lane = stencil cell), keep those whose box
        // some i reaches (warp-uniform loop over the chunk's atoms)
        int p_j0 = 0, p_jc = 0, p_js = -1;
        float p_sx = 0.f, p_sy = 0.f, p_sz = 0.f;
        float4 blo = make_float4(1e30f, 1e30f, 1e30f, 0.f), bhi = make_float4(-1e30f, -1e30f, -1e30f, 0.f);
        // HALF: own cell + the 13 forward cells (stencil order, device.py _stencil)
        if (lane < (HALF ? min(14, f.n_stencil) : f.n_stencil)) {
            const int ox = f.stencil[3 * lane], oy = f.stencil[3 * lane + 1], oz = f.stencil[3 * lane + 2];
            p_js = cell_probe(keys + hb, H, cx + ox, cy + oy, cz + oz);
            if (p_js >= 0) {
                p_sx = (float)ox * cellf; p_sy = (float)oy * cellf; p_sz = (float)oz * cellf;
                blo = cell_box[2 * (hb + p_js)]; bhi = cell_box[2 * (hb + p_js) + 1];
            }
        }
        __syncwarp();
        bool keep = false;
        for (int q = 0; q < ci_n; ++q) {
            const float4 r = ihi[q];
            const float px = r.x - p_sx, py = r.y - p_sy, pz = r.z - p_sz;
            const float gx = fmaxf(fmaxf(blo.x - px, px - bhi.x), 0.f);
            const float gy = fmaxf(fmaxf(blo.y - py, py - bhi.y), 0.f);
            const float gz = fmaxf(fmaxf(blo.z - pz, pz - bhi.z), 0.f);
            keep |= gx * gx + gy * gy + gz * gz <= pre2;
        }
        if (keep) { p_j0 = start[hb + p_js]; p_jc = cnt[hb + p_js]; }
        int p_end = p_jc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(FULL, p_end, o);
            if (lane >= o) p_end += v;
        }
        const int n_stream = __shfl_sync(FULL, p_end, 31);

        double ax = 0.0, ay = 0.0, az = 0.0, ee = 0.0, ev = 0.0;
        int ce = 0, cv = 0;
        for (int jb = SPLIT ? 32 * warp : 0; jb < n_stream; jb += SPLIT ? 32 * NW : 32) {
            const int nt = min(32, n_stream - jb);
            {
                const int e = jb + lane;
                int cs = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const int end = __shfl_sync(FULL, p_end, cs + step - 1);
                    if (end <= e) cs += step;
                }
                const int cend = __shfl_sync(FULL, p_end, cs), cj0 = __shfl_sync(FULL, p_j0, cs),
                          ccnt = __shfl_sync(FULL, p_jc, cs);
                const float ssx = __shfl_sync(FULL, p_sx, cs), ssy = __shfl_sync(FULL, p_sy, cs),
                            ssz = __shfl_sync(FULL, p_sz, cs);
                __syncwarp();
                if (lane < nt) {
                    const int kk = cj0 + (e - (cend - ccnt));
                    const size_t kj = nb + kk;
                    const float4 h = s_hi[kj];
                    int4 aux = s_aux[kj];
                    aux.w = kk;                     // sorted index (fp64 slow path)
                    J.hi[lane] = make_float4(h.x + ssx, h.y + ssy, h.z + ssz, 0.f);   // i's cell frame
                    J.lo[lane] = s_lo[kj];
                    J.par[lane] = s_par[kj];
                    J.aux[lane] = aux;
                }
                if (HALF) {
                    float4 *z = reinterpret_cast<float4 *>(&Jc_s[warp][0][0][0]);
#pragma unroll
                    for (int q = 0; q < 3 * 32 * 16 / 4 / 32; ++q) z[lane + 32 * q] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
                __syncwarp();
            }
            T fx = 0, fy = 0, fz = 0, fe = 0, fv = 0;
            if (HALF) {
                // each unordered pair once: own cell j after i (sorted order), forward
                // cells all; the force on j (-f) is kept per (j, owner) for this tile
                const int n_it = (nt + nph - 1) / nph;
                const int i_pos = ic + oi;              // i's position in its cell
                for (int kt = 0; kt < n_it; ++kt) {
                    const int t = ph + kt * nph;
                    // own-cell atoms lead the stream (stream positions < c, i_pos < c), so
                    // "j after i in the own cell, or j in a forward cell" is one compare
                    const bool live = own && t < nt && jb + t > i_pos;
                    const float4 hj = J.hi[t < nt ? t : 0];
                    const float dx = hi.x - hj.x, dy = hi.y - hj.y, dz = hi.z - hj.z;
                    const bool pass = live && dx * dx + dy * dy + dz * dz <= pre2;
                    if (!__any_sync(FULL, pass)) continue;
                    T out[5] = {0, 0, 0, 0, 0};
                    int pce = 0, pcv = 0;
                    if (pass) {
                        const int4 aj = J.aux[t];
                        double sd[5];
                        if (pair_eval<F64, T>(f, pc, hi, li, qi, ai, cm, hj, J.lo[t], J.par[t], aj, s_pos + ki,
                                              s_pos + nb + aj.w, status + b, out, pce, pcv, sd)) {
                            // exact path: fp64 forces straight into both atoms' fixed point
                            // (i gets +f, j gets -f; fj_combine adds the planes to every atom)
                            for (int q = 0; q < 3; ++q) {
                                fj_add(fj_fixed, fj_plane, 3 * (nb + ai.x) + q, sd[q]);
                                fj_add(fj_fixed, fj_plane, 3 * (nb + aj.x) + q, -sd[q]);
                            }
                            ee += sd[3]; ev += sd[4];
                        }
                    }
                    fx += out[0]; fy += out[1]; fz += out[2]; fe += out[3]; fv += out[4];
                    ce += pce; cv += pcv;
                    if (pass) {   // this lane's f on i for j = t (slot [t][oi]: one writer per
                        // tile); the flush subtracts, so j receives -f
                        Jc_s[warp][0][t][oi] = (float)out[0];
                        Jc_s[warp][1][t][oi] = (float)out[1];
                        Jc_s[warp][2][t][oi] = (float)out[2];
                    }
                }
                __syncwarp();
                // flush: the tile's j forces into the trajectory's two-level fixed point
                // (integer atomics: order-free, so the result is schedule-independent)
                if (lane < nt) {
                    double v[3];
#pragma unroll
                    for (int q = 0; q < 3; ++q) {   // owner slots in order: deterministic
                        const float4 *r = reinterpret_cast<const float4 *>(&Jc_s[warp][q][lane][0]);
                        float acc = 0.f;
                        for (int o4 = 0; o4 < (wi + 3) / 4; ++o4) {
                            const float4 c4 = r[o4];
                            acc -= c4.x; acc -= c4.y; acc -= c4.z; acc -= c4.w;   // (-a) + (-b) == -a - b
                        }
                        v[q] = (double)acc;
                    }
                    // planes: lo [B n 3], hi [B n 3], fp64 [B n 3] (the last two rarely touched)
                    for (int q = 0; q < 3; ++q) fj_add(fj_fixed, fj_plane, 3 * (nb + J.aux[lane].x) + q, v[q]);
                }
            } else {
                // this lane's prefilter hits over the tile (bit kt: j = ph + kt * nph), then
                // each lane walks its own hits in ascending order: the warp runs
                // max-over-lanes iterations, not one per j that any lane meets
                unsigned hits = 0;
                if (own)
                    for (int t = ph, kt = 0; t < nt; t += nph, ++kt) {
                        const float4 hj = J.hi[t];
                        const float dx = hi.x - hj.x, dy = hi.y - hj.y, dz = hi.z - hj.z;
                        if (dx * dx + dy * dy + dz * dz <= pre2) hits |= 1u << kt;
                    }
                while (hits) {
                    const int t = ph + (__ffs(hits) - 1) * nph;
                    hits &= hits - 1;
                    T out[5] = {0, 0, 0, 0, 0};
                    int pce = 0, pcv = 0;
                    const int4 aj = J.aux[t];
                    double sd[5];
                    if (pair_eval<F64, T>(f, pc, hi, li, qi, ai, cm, J.hi[t], J.lo[t], J.par[t], aj, s_pos + ki,
                                          s_pos + nb + aj.w, status + b, out, pce, pcv, sd)) {
                        ax += sd[0]; ay += sd[1]; az += sd[2]; ee += sd[3]; ev += sd[4];   // fp64 sums directly
                    }
                    fx += out[0]; fy += out[1]; fz += out[2]; fe += out[3]; fv += out[4];
                    ce += pce; cv += pcv;
                }
            }
            ax += (double)fx; ay += (double)fy; az += (double)fz;
            ee += (double)fe; ev += (double)fv;
            __syncwarp();
        }
        // combine the j phases of each owner (fixed xor tree: both partners get the same sum)
        for (int m = wi; m < 32; m <<= 1) {
            ax += __shfl_xor_sync(FULL, ax, m);
            ay += __shfl_xor_sync(FULL, ay, m);
            az += __shfl_xor_sync(FULL, az, m);
        }
        if (SPLIT) {
            // combine the warps' partial forces in warp order (deterministic)
            part[SPLIT ? warp : 0][0][lane] = ax;
            part[SPLIT ? warp : 0][1][lane] = ay;
            part[SPLIT ? warp : 0][2][lane] = az;
            __syncthreads();
            if (warp == 0 && own && ph == 0) {
                double sx = 0.0, sy = 0.0, sz = 0.0;
#pragma unroll
                for (int w = 0; w < (SPLIT ? NW : 1); ++w) {
                    sx += part[w][0][lane]; sy += part[w][1][lane]; sz += part[w][2][lane];
                }
                const size_t o = nb + ai.x;
                forces[3 * o] = sx; forces[3 * o + 1] = sy; forces[3 * o + 2] = sz;
                e_atom[2 * o] = 0.0; e_atom[2 * o + 1] = 0.0;
                pair_count[o] = 0;
            }
            __syncthreads();
        } else if (own && ph == 0) {
            const size_t o = nb + ai.x;
            forces[3 * o] = ax; forces[3 * o + 1] = ay; forces[3 * o + 2] = az;
            e_atom[2 * o] = 0.0; e_atom[2 * o + 1] = 0.0;
            pair_count[o] = 0;
        }
        if (HALF) { ee *= 2.0; ev *= 2.0; ce *= 2; cv *= 2; }   // pairs counted once: the reductions halve
        long long pcount = (long long)ce + ((long long)cv << 32);
        // chunk totals: fixed xor tree per warp, then warps in order, stored at the
        // chunk's first atom (chunks are a function of the positions: deterministic)
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            ee += __shfl_xor_sync(FULL, ee, d);
            ev += __shfl_xor_sync(FULL, ev, d);
            pcount += __shfl_xor_sync(FULL, pcount, d);
        }
        if (SPLIT) {
            if (lane == 0) { epart[warp][0] = ee; epart[warp][1] = ev; cpart[warp] = pcount; }
            __syncthreads();
            if (threadIdx.x == 0) {
                double te = 0.0, tv = 0.0;
                long long tc = 0;
                for (int w = 0; w < NW; ++w) { te += epart[w][0]; tv += epart[w][1]; tc += cpart[w]; }
                const size_t o = nb + s_aux[nb + s0 + ic].x;
                e_atom[2 * o] = te; e_atom[2 * o + 1] = tv;
                pair_count[o] = tc;
            }
        } else {
            __syncwarp();
            if (lane == 0) {
                const size_t o = nb + s_aux[nb + s0 + ic].x;
                e_atom[2 * o] = ee; e_atom[2 * o + 1] = ev;
                pair_count[o] = pcount;
            }
        }
    }
}

// forces += the half-list kernel's j-side fixed point, which is then cleared
// (thread = one force component: coalesced over the [B][n][3] forces)
__global__ void fj_combine_kernel(int B, int n, long long *__restrict__ fj, double *__restrict__ forces,
                                  const kf_status_t *status) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= 3LL * B * n) return;
    const long long a = gid / 3;
    const int q = (int)(gid - 3 * a);
    if (status[a / n].done) return;
    long long *p = fj + 3 * a;
    const long long plane = 3LL * B * n;
    const long long lo = p[q], hi = p[plane + q];
    double *big = reinterpret_cast<double *>(fj + 2 * plane) + 3 * a + q;
    const double bg = *big;
    if (lo || hi || bg != 0.0) {
        forces[gid] += ((double)hi * FJ_HI + (double)lo * FJ_LO) + bg;
        if (lo) p[q] = 0;             // clear only what was written (the hi and fp64 planes
        if (hi) p[plane + q] = 0;     // are rarely touched: no 8-byte store per component)
        if (bg != 0.0) *big = 0.0;
    }
}

// On error only: smallest (i, j), i < j, among pairs at the minimum distance.
__global__ void clash_report_kernel(kf_field_t f, int B, int n, const unsigned long long *__restrict__ keys,
                                    const int32_t *__restrict__ cnt, const int32_t *__restrict__ start,
                                    const int32_t *__restrict__ atom_slot, const double4 *__restrict__ s_pos,
                                    const int4 *__restrict__ s_aux, const double *__restrict__ pos,
                                    kf_status_t *status) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (long long)B * n) return;
    const int b = (int)(gid / n), i = (int)(gid % n);
    if (status[b].error != KF_ERR_CLASH) return;
    const uint32_t H = 1u << f.hash_bits;
    const size_t hb = (size_t)b * H, nb = (size_t)b * n;
    int cx, cy, cz;
    unpack_cell((long long)keys[hb + atom_slot[gid]], cx, cy, cz);
    const double xi = pos[3 * gid], yi = pos[3 * gid + 1], zi = pos[3 * gid + 2];
    const unsigned long long target = status[b].dmin_bits;
    for (int s = 0; s < f.n_stencil; ++s) {
        const int js = cell_probe(keys + hb, H, cx + f.stencil[3 * s], cy + f.stencil[3 * s + 1],
                                  cz + f.stencil[3 * s + 2]);
        if (js < 0) continue;
        for (int k = start[hb + js]; k < start[hb + js] + cnt[hb + js]; ++k) {
            const int j = s_aux[nb + k].x;
            if (j <= i) continue;
            const double4 pj = s_pos[nb + k];
            const double d2 = d2_einsum(xsub(xi, pj.x), xsub(yi, pj.y), xsub(zi, pj.z));
            if (d2 > f.cut_pair2) continue;
            if ((unsigned long long)__double_as_longlong(sqrt(d2)) == target)
                atomicMin(reinterpret_cast<unsigned long long *>(&status[b].clash_key),
                          ((unsigned long long)i << 32) | (unsigned)j);
        }
    }
}

int g_sms = 0;

// Persistent grid: every CTA the SMs can hold (occupancy API), per kernel.
template <typename K>
int resident_grid(K kern, int threads, size_t dyn) {
    struct Entry { const void *k; size_t dyn; int grid; };
    static Entry cache[16];
    static int n_cache = 0;
    for (int e = 0; e < n_cache; ++e)
        if (cache[e].k == (const void *)kern && cache[e].dyn == dyn) return cache[e].grid;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, dyn);
    const int grid = g_sms * (per_sm > 0 ? per_sm : 1);
    if (n_cache < 16) cache[n_cache++] = Entry{(const void *)kern, dyn, grid};
    return grid;
}

}  // namespace

int kf_cluster_path(const kf_field_t *f, const kf_batch_t *w, int n);
int kf_cluster_pairs_launch(const kf_field_t *f, kf_batch_t *w, int n, cudaStream_t s, int plane_b);
int kf_cluster_clash_report_launch(const kf_field_t *f, kf_batch_t *w, int n, cudaStream_t s);

// The pair kernel a launch of (f, w, n) selects: 0 compacted list (fp64 pair math),
// 1 dense lanes full list, 2 dense lanes half list, 3 cluster pairs (kf_cluster.cu).
static int pair_variant(const kf_field_t *f, const kf_batch_t *w, int n) {
    if (kf_cluster_path(f, w, n)) return 3;
    static long long split_below = -1;
    if (split_below < 0) {
        const char *env = getenv("KFB200_PAIR_SPLIT_BELOW");
        split_below = env ? atoll(env) : 40000;
    }
    static int env_variant = -1;
    if (env_variant < 0) {
        const char *env = getenv("KFB200_PAIR_KERNEL");
        env_variant = env ? atoi(env) : 0;
    }
    const bool split = (long long)w->B * n < split_below;
    int variant = env_variant ? env_variant : (f->precision ? 1 : split ? 2 : 3);
    const int chunk = kf_pair_chunk(w->B, n, w->pair_chunk, f->precision);
    if (variant == 3 && (f->precision || !w->pair_fj || chunk > 16)) variant = f->precision ? 1 : 2;
    return variant - 1;
}

extern "C" int kf_pair_kernel_kind(const kf_field_t *f, const kf_batch_t *w, int n) {
    return pair_variant(f, w, n);
}

int kf_pairs_launch(const kf_field_t *f, kf_batch_t *w, int n, cudaStream_t s, int plane_b) {
    // ensembles with fp32 pair math: the cluster-pair kernel (kf_cluster.cu)
    if (kf_cluster_path(f, w, n)) return kf_cluster_pairs_launch(f, w, n, s, plane_b);
    if (g_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    KF_CUDA(cudaMemsetAsync(w->work, 0, sizeof(int32_t), s), "memset work");
    // one CTA per cell when the whole batch is small (latency), one warp per cell otherwise;
    // KFB200_PAIR_SPLIT_BELOW overrides the crossover (atoms per launch)
    static long long split_below = -1;
    if (split_below < 0) {
        const char *env = getenv("KFB200_PAIR_SPLIT_BELOW");
        split_below = env ? atoll(env) : 40000;
    }
    const bool split = (long long)w->B * n < split_below;
    // KFB200_PAIR_KERNEL: 1 = compacted pair list, 2 = dense lanes (full list),
    // 3 = dense lanes, half list (Newton's third law; j-side forces in integer
    // fixed point).  Default: half list for fp32 pair math on ensembles, full list
    // for small launches, compacted for fp64 (its pair body is long enough that
    // full lanes pay for the compaction).
    static int env_variant = -1;
    if (env_variant < 0) {
        const char *env = getenv("KFB200_PAIR_KERNEL");
        env_variant = env ? atoi(env) : 0;
    }
    // (the half list wins for ensembles; a lone chain's latency-bound CTA-per-item
    // pass does better on the full list without the fixed-point pass)
    int variant = env_variant ? env_variant : (f->precision ? 1 : split ? 2 : 3);
    const int chunk = kf_pair_chunk(w->B, n, w->pair_chunk, f->precision);
    // the half list needs its fixed-point buffer and chunks of <= 16 atoms
    if (variant == 3 && (f->precision || !w->pair_fj || chunk > 16)) variant = f->precision ? 1 : 2;
    const int nw = split ? SPLIT_WARPS : PAIR_WARPS;
    static bool opted = false;
    if (!opted) {
        for (auto k : {pair_kernel<true, true>, pair_kernel<true, false>, pair_kernel<false, true>,
                       pair_kernel<false, false>})
            KF_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024), "pair smem");
        opted = true;
    }
    PairConst pc;
    for (int q = 0; q < 4; ++q) {
        pc.we[q] = (float)(f->uniform_weights ? f->uniform_value : f->w_elec[q]);
        pc.wv[q] = (float)(f->uniform_weights ? f->uniform_value : f->w_vdw[q]);
    }
    pc.pre2 = (float)(f->cut_pair2 + 1e-2);
    pc.cut2 = (float)f->cut_pair2; pc.tv2 = (float)f->thr_vdw2; pc.te2 = (float)f->thr_elec2;
    pc.kap_inv = f->dielectric_const ? (float)(1.0 / f->kappa) : 1.0f;
    pc.cell = (float)f->cell;
    static float f64_below = -1.f;   // KFB200_PAIR_F64_BELOW (A): fp64 radius of the fp32 mode
    if (f64_below < 0.f) {
        const char *env = getenv("KFB200_PAIR_F64_BELOW");
        f64_below = env ? (float)atof(env) : 1.0f;
    }
    pc.f64_d2 = f64_below * f64_below;
    pc.dconst = f->dielectric_const; pc.uniform = f->uniform_weights;
    pc.te_is_cut = fabs(f->thr_elec2 - f->cut_pair2) < 1e-6 ? 1 : 0;
#define KF_PAIR_ARGS                                                                                          \
    *f, pc, w->B, n, chunk, w->cell_key, w->cell_cnt, w->cell_start, w->occ, w->occ_count, w->chunk_pre, w->item_cell, \
        w->chunk_offset, reinterpret_cast<const float4 *>(w->s_hi), reinterpret_cast<const float4 *>(w->s_lo), \
        reinterpret_cast<const double4 *>(w->s_pos), reinterpret_cast<const float4 *>(w->s_par),              \
        reinterpret_cast<const int4 *>(w->s_aux), reinterpret_cast<const int4 *>(w->s_tree),                  \
        reinterpret_cast<const float4 *>(w->cell_box), w->work, w->forces, w->e_atom, w->pair_count, w->status
    if (variant == 1) {
        const size_t dyn = (size_t)nw * (f->precision ? sizeof(WarpSmem<double>) : sizeof(WarpSmem<float>));
        auto kern = f->precision ? (split ? pair_kernel<true, true> : pair_kernel<true, false>)
                                 : (split ? pair_kernel<false, true> : pair_kernel<false, false>);
        kern<<<resident_grid(kern, nw * 32, dyn), nw * 32, dyn, s>>>(KF_PAIR_ARGS);
    } else {
        const bool half = variant == 3;
        auto kern = half ? (split ? pair_dense_kernel<false, true, true> : pair_dense_kernel<false, false, true>)
                         : f->precision ? (split ? pair_dense_kernel<true, true, false> : pair_dense_kernel<true, false, false>)
                                        : (split ? pair_dense_kernel<false, true, false> : pair_dense_kernel<false, false, false>);
        (void)kf_launch(w->B < KF_PDL_B, kern, dim3(resident_grid(kern, nw * 32, 0)), dim3(nw * 32), 0, s, KF_PAIR_ARGS,
                        w->pair_fj);
        if (half) {
            KF_LAUNCH_CHECK("pair_kernel");
            const long long total = 3LL * w->B * n;
            fj_combine_kernel<<<kf_blocks(total, 256), 256, 0, s>>>(w->B, n, w->pair_fj, w->forces, w->status);
        }
    }
#undef KF_PAIR_ARGS
    KF_LAUNCH_CHECK("pair_kernel");
    return 0;
}

int kf_clash_report_launch(const kf_field_t *f, kf_batch_t *w, int n, cudaStream_t s) {
    if (kf_cluster_path(f, w, n)) return kf_cluster_clash_report_launch(f, w, n, s);
    const long long total = (long long)w->B * n;
    clash_report_kernel<<<kf_blocks(total, 128), 128, 0, s>>>(
        *f, w->B, n, w->cell_key, w->cell_cnt, w->cell_start, w->atom_slot,
        reinterpret_cast<const double4 *>(w->s_pos), reinterpret_cast<const int4 *>(w->s_aux), w->pos, w->status);
    KF_LAUNCH_CHECK("clash_report_kernel");
    return 0;
}
