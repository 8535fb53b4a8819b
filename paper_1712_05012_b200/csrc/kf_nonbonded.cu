// Nonbonded elec + vdW pair kernel (K3) with the cut-off filter (K2), the
// 1-2/1-3/1-4 classifier and the steric-clash guard fused in.
//
// Reference: Field.evaluate's force phase (/root/reference/pkg/src/kinefold/
// kcm.py:110-127) = extract_pairs (forcefield.py:81-89 -> spatial.py:233-241),
// TreeWeights.weights_for (topology.py:153-195), elec/vdw_pair_quantities
// (forcefield.py:98-113) and the bincount scatter (forcefield.py:162-172).
//
// Work: one warp per occupied 9 A cell (dynamic work counter over the cells of
// all trajectories); the cell's atoms (<= 32 per pass) are the warp's i-tile.
// For each of the 27 neighbour cells that some lane can reach (per-lane
// distance to the cell's bounding box, warp vote) the warp stages 32-atom
// j-tiles in shared memory and runs two stages:
//   1. prefilter: each lane tests its i against the tile in fp32 from
//      cell-centre offsets into a 32-bit mask (band 1e-2 A^2 around cut^2);
//   2. compacted pairs: the set bits of all lanes are dealt out one pair per
//      lane (warp scan + __fns), so every lane does useful pair work; each
//      pair gets its difference vector from the hi/lo fp32 offset pairs
//      (fp64-accurate), decides membership exactly as the reference
//      (d2 = (dx*dx + dz*dz) + dy*dy in fp64 vs max(elec, vdw)^2, and
//      sqrt(d2) <= cut per term) — recomputed from the fp64 positions only in
//      a 1e-3 A^2 band around each threshold — and evaluates energy and
//      force in fp32; pairs under 1 A take the reference's fp64 formulas.
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
constexpr int PAIR_WARPS = 4;        // warps per CTA, warp-per-cell variant
constexpr int SPLIT_WARPS = 4;       // warps per CTA (one cell), split variant
constexpr unsigned FULL = 0xffffffffu;

struct Tile {
    float4 hi[32];
    float4 lo[32];
    float4 par[32];
    int4 aux[32];
};

constexpr int RES_BATCH = 128;

template <typename T>
struct WarpSmem {
    Tile J;
    T res[RES_BATCH][3];       // per-pair forces of the current batch of the tile's list
    unsigned short list[1024]; // candidate (owner << 5 | t) pairs of the tile, owner-major
};

struct Acc {
    double fx, fy, fz, ee, ev;
    long long cnt;   // elec-cutoff partners (low 32 bits) | vdW-cutoff partners << 32
};

// One pair in fp64 (the reference's formulas, forcefield.py:98-113, with the
// powers written as products): used below 1 A, and for every pair in the
// fp64 precision mode.
template <typename T>
KF_DEV void pair_fp64(const kf_field_t &f, int i, int j, double d2, double dx, double dy, double dz,
                      double we, double wv, bool ke, bool kv, T *out) {
    const double d = sqrt(d2);
    const double inv_d = 1.0 / d;
    double mag = 0.0, ee = 0.0, ev = 0.0;
    if (ke) {
        const double num = COULOMB_K * we * f.q[i] * f.q[j];
        ee = f.dielectric_const ? num * inv_d / f.kappa : num * inv_d * inv_d;   // num / (kappa d)
        mag += ee * inv_d;                                                       // num / (kappa d^2)
    }
    if (kv) {
        const double eps = sqrt(f.eps[i] * f.eps[j]);
        const double r = (f.R[i] + f.R[j]) * inv_d;
        const double r2 = r * r, r6 = r2 * r2 * r2;
        ev = wv * eps * (r6 * r6 - 2.0 * r6);
        mag += 12.0 * wv * eps * (r6 * r6 - r6) * inv_d;
    }
    const double g = mag * inv_d;
    out[0] = (T)(g * dx); out[1] = (T)(g * dy); out[2] = (T)(g * dz);
    out[3] = (T)ee; out[4] = (T)ev;
}

// Everything the exact / fp64 pair path needs, kept out of the kernel's
// register allocation (the path runs for pairs within 1e-3 A^2 of a cut-off,
// below 1 A, or always in fp64 mode).
struct SlowArgs {
    const double *q, *R, *eps;
    double kappa, cut2, te2, tv2, wel[4], wvd[4];
    int dconst;
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
__device__ __noinline__ void slow_pair(bool f64, const SlowArgs &A, const double4 *pi_, const double4 *pj_, int i,
                                       int j, int cls, T *out, int *pce, int *pcv, kf_status_t *st) {
    const double4 p_i = *pi_, p_j = *pj_;
    const double dx = xsub(p_i.x, p_j.x), dy = xsub(p_i.y, p_j.y), dz = xsub(p_i.z, p_j.z);
    const double d2 = d2_einsum(dx, dy, dz);
    if (d2 > A.cut2) return;
    const bool ke = d2 <= A.te2, kv = d2 <= A.tv2;
    *pce = ke; *pcv = kv;
    const double we = A.wel[cls - 1], wv = A.wvd[cls - 1];
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
        const double num = COULOMB_K * we * A.q[i] * A.q[j];
        ee = A.dconst ? num * inv_d / A.kappa : num * inv_d * inv_d;   // num / (kappa d)
        mag += ee * inv_d;                                              // num / (kappa d^2)
    }
    if (kv) {
        const double eps = sqrt(A.eps[i] * A.eps[j]);
        const double r = (A.R[i] + A.R[j]) * inv_d;
        const double r2 = r * r, r6 = r2 * r2 * r2;
        ev = wv * eps * (r6 * r6 - 2.0 * r6);
        mag += 12.0 * wv * eps * (r6 * r6 - r6) * inv_d;
    }
    const double g = mag * inv_d;
    out[0] = (T)(g * dx); out[1] = (T)(g * dy); out[2] = (T)(g * dz);
    out[3] = (T)ee; out[4] = (T)ev;
    (void)f64;
}

#ifndef PAIR_MINB
#define PAIR_MINB 3
#endif
// F64 = false: fp32 pair math (the north-star configuration); true: fp64
// pair math and fp64 per-tile sums (strict trajectory parity mode).
// SPLIT = true: one CTA per cell, its 4 warps split the 27 neighbour cells
// (short per-cell latency: single trajectories); false: one warp per cell
// (throughput: ensembles).
template <bool F64, bool SPLIT>
__global__ void __launch_bounds__((SPLIT ? SPLIT_WARPS : PAIR_WARPS) * 32, SPLIT ? 1 : 4)
pair_kernel(kf_field_t f, int B, int n, const unsigned long long *__restrict__ keys,
            const int32_t *__restrict__ cnt, const int32_t *__restrict__ start, const int32_t *__restrict__ occ,
            const int32_t *__restrict__ occ_count, const int32_t *__restrict__ chunk_pre,
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
    const float cellf = (float)f.cell;
    const float pre2 = (float)(f.cut_pair2 + 1e-2);
    const float cut2f = (float)f.cut_pair2, tvf = (float)f.thr_vdw2, tef = (float)f.thr_elec2;
    const float band = 1e-3f;
    const float kap_inv = f.dielectric_const ? (float)(1.0 / f.kappa) : 1.0f;
    float wf[8];
    for (int q = 0; q < 4; ++q) {
        wf[q] = f.uniform_weights ? (float)f.uniform_value : (float)f.w_elec[q];
        wf[4 + q] = f.uniform_weights ? (float)f.uniform_value : (float)f.w_vdw[q];
    }
    SlowArgs fx64;
    fx64.q = f.q; fx64.R = f.R; fx64.eps = f.eps;
    fx64.kappa = f.kappa; fx64.cut2 = f.cut_pair2; fx64.te2 = f.thr_elec2; fx64.tv2 = f.thr_vdw2;
    fx64.dconst = f.dielectric_const;
    for (int q = 0; q < 4; ++q) {
        fx64.wel[q] = f.uniform_weights ? f.uniform_value : f.w_elec[q];
        fx64.wvd[q] = f.uniform_weights ? f.uniform_value : f.w_vdw[q];
    }

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
        int klo = 0, khi = occ_count[b] - 1;          // last k with chunk_pre[k] <= local
        while (klo < khi) {
            const int mid = (klo + khi + 1) >> 1;
            if (chunk_pre[hb + mid] <= local) klo = mid; else khi = mid - 1;
        }
        const int slot = occ[hb + klo];
        const int ic = (local - chunk_pre[hb + klo]) << 5;
        int cx, cy, cz;
        unpack_cell((long long)keys[hb + slot], cx, cy, cz);
        const int s0 = start[hb + slot], c = cnt[hb + slot];
        double ee = 0.0, ev = 0.0;   // cell totals (per computing lane)
        long long pcount = 0;
        {
            const int ci_n = min(32, c - ic);
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
            const float4 hi_i = I.hi[valid ? lane : 0];
            Acc a = {0.0, 0.0, 0.0, 0.0, 0.0, 0};

            // the 27 neighbour cells are dealt to the warps round-robin; each warp
            // keeps per-owner fp64 sums over its cells in a fixed order
            // probe all neighbour cells at once (lane s <-> stencil cell s): one
            // round of table / start / count / box loads instead of 27 serial ones
            int p_js = -1, p_j0 = 0, p_jc = 0;
            float4 p_lo = make_float4(0.f, 0.f, 0.f, 0.f), p_hi = p_lo;
            if (lane < f.n_stencil) {
                p_js = cell_probe(keys + hb, H, cx + f.stencil[3 * lane], cy + f.stencil[3 * lane + 1],
                                  cz + f.stencil[3 * lane + 2]);
                if (p_js >= 0) {
                    p_j0 = start[hb + p_js]; p_jc = cnt[hb + p_js];
                    p_lo = cell_box[2 * (hb + p_js)]; p_hi = cell_box[2 * (hb + p_js) + 1];
                }
            }
            for (int s = SPLIT ? warp : 0; s < f.n_stencil; s += SPLIT ? NW : 1) {
                const int js = __shfl_sync(FULL, p_js, s);
                if (js < 0) continue;
                const int ox = f.stencil[3 * s], oy = f.stencil[3 * s + 1], oz = f.stencil[3 * s + 2];
                // i in the neighbour cell's frame; skip the cell unless some lane reaches its box
                const float sx = (float)ox * cellf, sy = (float)oy * cellf, sz = (float)oz * cellf;
                const float px = hi_i.x - sx, py = hi_i.y - sy, pz = hi_i.z - sz;
                const float blx = __shfl_sync(FULL, p_lo.x, s), bly = __shfl_sync(FULL, p_lo.y, s),
                            blz = __shfl_sync(FULL, p_lo.z, s);
                const float bhx = __shfl_sync(FULL, p_hi.x, s), bhy = __shfl_sync(FULL, p_hi.y, s),
                            bhz = __shfl_sync(FULL, p_hi.z, s);
                const float gx = fmaxf(fmaxf(blx - px, px - bhx), 0.f);
                const float gy = fmaxf(fmaxf(bly - py, py - bhy), 0.f);
                const float gz = fmaxf(fmaxf(blz - pz, pz - bhz), 0.f);
                const bool need = valid && gx * gx + gy * gy + gz * gz <= pre2;
                if (!__any_sync(FULL, need)) continue;
                const int j0 = __shfl_sync(FULL, p_j0, s), jc = __shfl_sync(FULL, p_jc, s);
                for (int jb = 0; jb < jc; jb += 32) {
                    const int nt = min(32, jc - jb);
                    __syncwarp();
                    if (lane < nt) {
                        const size_t kj = nb + j0 + jb + lane;
                        S.J.hi[lane] = s_hi[kj];
                        S.J.lo[lane] = s_lo[kj];
                        S.J.par[lane] = s_par[kj];
                        S.J.aux[lane] = s_aux[kj];
                    }
                    __syncwarp();
                    // ---- stage 1: fp32 prefilter into a mask
                    unsigned mask = 0u;
                    if (need) {
                        for (int t = 0; t < nt; ++t) {
                            const float4 r = S.J.hi[t];
                            const float dx = px - r.x, dy = py - r.y, dz = pz - r.z;
                            mask |= (dx * dx + dy * dy + dz * dz <= pre2 ? 1u : 0u) << t;
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
                            const int i = ai.x, j = aj.x;
                            const float4 hi = I.hi[o], li = I.lo[o], hj = S.J.hi[t], lj = S.J.lo[t];
                            const float dxf = ((hi.x - hj.x) - sx) + (li.x - lj.x);
                            const float dyf = ((hi.y - hj.y) - sy) + (li.y - lj.y);
                            const float dzf = ((hi.z - hj.z) - sz) + (li.z - lj.z);
                            const float d2f = dxf * dxf + dyf * dyf + dzf * dzf;
                            if (i != j && d2f <= cut2f + band) {
                                // static class window: 2-bit codes for j - i in [-32, 32)
                                int cls = 4;
                                if (!f.uniform_weights) {
                                    const int off = j - i + 32;
                                    if ((unsigned)off < 64u) {
                                        const int4 cm = itree[o];
                                        const unsigned wd = off < 32 ? (off < 16 ? cm.x : cm.y)
                                                                     : (off < 48 ? cm.z : cm.w);
                                        cls = 4 - (int)((wd >> (2 * (off & 15))) & 3u);
                                    } else if (ai.w != 0 && aj.z != 0 && abs(ai.y - aj.y) <= 1) {
                                        cls = slow_class(f.tparent, f.tgp, f.tggp, f.tres, f.tchain, i, j);
                                    }
                                }
                                const float we = cls == 4 ? wf[3] : cls == 3 ? wf[2] : cls == 2 ? wf[1] : wf[0];
                                const float wv = cls == 4 ? wf[7] : cls == 3 ? wf[6] : cls == 2 ? wf[5] : wf[4];
                                const bool exact = F64 || fabsf(d2f - cut2f) <= band || fabsf(d2f - tvf) <= band ||
                                                   fabsf(d2f - tef) <= band || d2f < 1.0f;
                                if (exact) {
                                    slow_pair<T>(F64, fx64, s_pos + nb + s0 + ic + o, s_pos + nb + j0 + jb + t, i, j,
                                                 cls, out, &pce, &pcv, status + b);
                                } else if (d2f <= cut2f) {
                                    const bool ke = d2f <= tef, kv = d2f <= tvf;
                                    pce = ke; pcv = kv;
                                    const float4 qi = I.par[o], qj = S.J.par[t];
                                    const float inv_r = rsqrtf(d2f);
                                    const float inv_r2 = inv_r * inv_r;
                                    float g = 0.f;
                                    if (ke) {
                                        // kappa = d: E = K w qi qj / d^2; constant: E = K w qi qj / (kappa d);
                                        // |F| / d = E / d^2 in both cases
                                        const float qq = (float)COULOMB_K * qi.x * qj.x * we;
                                        const float e = f.dielectric_const ? qq * kap_inv * inv_r : qq * inv_r2;
                                        out[3] = e;
                                        g += e * inv_r2;
                                    }
                                    if (kv) {
                                        const float weps = wv * qi.z * qj.z;
                                        const float D = qi.y + qj.y;
                                        const float sr = D * D * inv_r2;
                                        const float s3 = sr * sr * sr;
                                        const float s6 = s3 * s3;
                                        out[4] = weps * (s6 - 2.f * s3);
                                        g += 12.f * weps * (s6 - s3) * inv_r2;
                                    }
                                    out[0] = g * dxf; out[1] = g * dyf; out[2] = g * dzf;
                                }
                            }
                        }
                        const long long pc = (long long)pce + ((long long)pcv << 32);
                        // energies and counts only enter per-cell totals: the computing lane keeps them
                        fe += out[3]; fv += out[4];
                        a.cnt += pc;
                        if (act) { S.res[k0 + lane][0] = out[0]; S.res[k0 + lane][1] = out[1]; S.res[k0 + lane][2] = out[2]; }
                      }
                      __syncwarp();
                      // each owner sums its contiguous range of the list in order (deterministic)
                      const int lo_k = max(excl - base, 0), hi_k = min(incl - base, nbat);
                      for (int q = lo_k; q < hi_k; ++q) { fx += S.res[q][0]; fy += S.res[q][1]; fz += S.res[q][2]; }
                      __syncwarp();
                    }
                    a.fx += (double)fx; a.fy += (double)fy; a.fz += (double)fz;
                    a.ee += (double)fe; a.ev += (double)fv;
                }
            }
            ee += a.ee; ev += a.ev; pcount += a.cnt;
            if (SPLIT) {
                // combine the warps' partial forces in warp order (deterministic)
                part[SPLIT ? warp : 0][0][lane] = a.fx;
                part[SPLIT ? warp : 0][1][lane] = a.fy;
                part[SPLIT ? warp : 0][2][lane] = a.fz;
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
                forces[3 * o] = a.fx; forces[3 * o + 1] = a.fy; forces[3 * o + 2] = a.fz;
                e_atom[2 * o] = 0.0; e_atom[2 * o + 1] = 0.0;
                pair_count[o] = 0;
            }
        }
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

int g_pair_grid = 0;

}  // namespace

int kf_pairs_launch(const kf_field_t *f, kf_batch_t *w, int n, cudaStream_t s) {
    if (g_pair_grid == 0) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        g_pair_grid = sms * 4;
    }
    KF_CUDA(cudaMemsetAsync(w->work, 0, sizeof(int32_t), s), "memset work");
    // one CTA per cell when the whole batch is small (latency), one warp per cell otherwise;
    // KFB200_PAIR_SPLIT_BELOW overrides the crossover (atoms per launch)
    static long long split_below = -1;
    if (split_below < 0) {
        const char *env = getenv("KFB200_PAIR_SPLIT_BELOW");
        split_below = env ? atoll(env) : 200000;
    }
    const bool split = (long long)w->B * n < split_below;
    auto kern = f->precision ? (split ? pair_kernel<true, true> : pair_kernel<true, false>)
                             : (split ? pair_kernel<false, true> : pair_kernel<false, false>);
    const int nw = split ? SPLIT_WARPS : PAIR_WARPS;
    const size_t dyn = (size_t)nw * (f->precision ? sizeof(WarpSmem<double>) : sizeof(WarpSmem<float>));
    static bool opted = false;
    if (!opted) {
        for (auto k : {pair_kernel<true, true>, pair_kernel<true, false>, pair_kernel<false, true>,
                       pair_kernel<false, false>})
            KF_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024), "pair smem");
        opted = true;
    }
    kern<<<split ? g_pair_grid / 2 : g_pair_grid, nw * 32, dyn, s>>>(
        *f, w->B, n, w->cell_key, w->cell_cnt, w->cell_start, w->occ, w->occ_count, w->chunk_pre, w->chunk_offset,
        reinterpret_cast<const float4 *>(w->s_hi), reinterpret_cast<const float4 *>(w->s_lo),
        reinterpret_cast<const double4 *>(w->s_pos), reinterpret_cast<const float4 *>(w->s_par),
        reinterpret_cast<const int4 *>(w->s_aux), reinterpret_cast<const int4 *>(w->s_tree),
        reinterpret_cast<const float4 *>(w->cell_box), w->work, w->forces, w->e_atom, w->pair_count,
        w->status);
    KF_LAUNCH_CHECK("pair_kernel");
    return 0;
}

int kf_clash_report_launch(const kf_field_t *f, kf_batch_t *w, int n, cudaStream_t s) {
    const long long total = (long long)w->B * n;
    clash_report_kernel<<<kf_blocks(total, 128), 128, 0, s>>>(
        *f, w->B, n, w->cell_key, w->cell_cnt, w->cell_start, w->atom_slot,
        reinterpret_cast<const double4 *>(w->s_pos), reinterpret_cast<const int4 *>(w->s_aux), w->pos, w->status);
    KF_LAUNCH_CHECK("clash_report_kernel");
    return 0;
}
