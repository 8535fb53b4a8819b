// Nonbonded elec + vdW pair kernel (K3) with the cut-off filter (K2), the
// 1-2/1-3/1-4 classifier and the steric-clash guard fused in.
//
// Reference: Field.evaluate's force phase (/root/reference/pkg/src/kinefold/
// kcm.py:110-127) = extract_pairs (forcefield.py:81-89 -> spatial.py:233-241),
// TreeWeights.weights_for (topology.py:153-195), elec/vdw_pair_quantities
// (forcefield.py:98-113) and the bincount scatter (forcefield.py:162-172).
//
// Layout: one warp per occupied 9 A cell (persistent grid over the work list
// of all trajectories); lanes own the cell's atoms.  For each of the 27
// neighbour cells the warp stages 32-atom j-tiles in shared memory (one
// coalesced load per lane, then broadcast reads) and each lane
//   1. prefilters the tile in fp32 from cell-centre offsets (no absolute
//      coordinates, so |error| < 1e-5 A^2, far inside a 1e-2 A^2 band), into
//      a bit mask;
//   2. walks the mask: exact reference membership in fp64 — d2 in einsum
//      order (dx*dx + dz*dz) + dy*dy vs max(elec, vdw)^2, and sqrt(d2) <= cut
//      per term via the equivalent d2 thresholds — then the pair energy and
//      force in fp32 from the fp64 difference vector, fp64 per-atom sums
//      (pairs closer than 0.1 A take the reference's fp64 formulas).
// Both directions of each unordered pair are evaluated by their owners
// ("full list"): no atomics, fixed accumulation order, run-to-run bitwise
// deterministic.
#include "kf_common.cuh"

namespace {

constexpr double COULOMB_K = 332.06;
constexpr double MIN_DISTANCE = 1e-6;
constexpr double FP64_BELOW_D2 = 1e-2;
constexpr int PAIR_WARPS = 4;

struct JTile {
    float4 rel[32];
    double4 pos[32];
    float4 par[32];
    int4 aux[32];
};

struct Acc {
    double fx, fy, fz, ee, ev;
    int cnt;   // elec-cutoff partners (low 16 bits) | vdW-cutoff partners << 16
};

// Reference fp64 formulas for one pair (used at d < 0.1 A).
KF_DEV void pair_fp64(const kf_field_t &f, int i, int j, double d2, double dx, double dy, double dz,
                      double we, double wv, bool ke, bool kv, Acc &a) {
    const double d = sqrt(d2);
    double mag = 0.0;
    if (ke) {
        const double kap = f.dielectric_const ? f.kappa : d;
        const double num = COULOMB_K * we * f.q[i] * f.q[j];
        a.ee += num / (kap * d);
        mag += num / (kap * d * d);
    }
    if (kv) {
        const double eps = sqrt(f.eps[i] * f.eps[j]);
        const double dd = f.R[i] + f.R[j];
        const double dd6 = pow(dd, 6.0), d6 = pow(d, 6.0);
        const double ratio6 = dd6 / d6;
        a.ev += wv * eps * (ratio6 * ratio6 - 2.0 * ratio6);
        mag += 12.0 * wv * eps * (pow(dd, 12.0) / pow(d, 13.0) - dd6 / pow(d, 7.0));
    }
    const double g = mag / d;
    a.fx += g * dx; a.fy += g * dy; a.fz += g * dz;
}

__global__ void __launch_bounds__(PAIR_WARPS * 32)
pair_kernel(kf_field_t f, int B, int n, const unsigned long long *__restrict__ keys,
            const int32_t *__restrict__ cnt, const int32_t *__restrict__ start, const int32_t *__restrict__ occ,
            const int32_t *__restrict__ occ_offset, const float4 *__restrict__ s_rel,
            const double4 *__restrict__ s_pos, const float4 *__restrict__ s_par, const int4 *__restrict__ s_aux,
            double *__restrict__ forces, double *__restrict__ e_atom, int32_t *__restrict__ pair_count,
            kf_status_t *status) {
    __shared__ JTile tiles[PAIR_WARPS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    JTile &T = tiles[warp];
    const uint32_t H = 1u << f.hash_bits;
    const int total = occ_offset[B];
    const float cellf = (float)f.cell;
    const float pre2 = (float)(f.cut_pair2 + 1e-2);
    const float kap_inv = f.dielectric_const ? (float)(1.0 / f.kappa) : 1.0f;

    for (int item = blockIdx.x * PAIR_WARPS + warp; item < total; item += gridDim.x * PAIR_WARPS) {
        const int b = item_owner(occ_offset, B, item);
        const size_t hb = (size_t)b * H, nb = (size_t)b * n;
        const int slot = occ[hb + (item - occ_offset[b])];
        int cx, cy, cz;
        unpack_cell((long long)keys[hb + slot], cx, cy, cz);
        const int s0 = start[hb + slot], c = cnt[hb + slot];
        for (int ic = 0; ic < c; ic += 32) {
            const bool valid = ic + lane < c;
            const size_t ki = nb + s0 + ic + (valid ? lane : 0);
            const float4 ri = s_rel[ki];
            const double4 pi4 = s_pos[ki];
            const float4 qi4 = s_par[ki];
            const int4 ai = s_aux[ki];
            const int i = ai.x;
            int pi = -1, gpi = -1, ggi = -1;
            const bool ci = !f.uniform_weights && ai.z != 0;
            if (ci) { pi = f.tparent[i]; gpi = f.tgp[i]; ggi = f.tggp[i]; }
            const float qi = qi4.x * (float)COULOMB_K;
            Acc a = {0.0, 0.0, 0.0, 0.0, 0.0, 0};

            for (int s = 0; s < f.n_stencil; ++s) {
                const int ox = f.stencil[3 * s], oy = f.stencil[3 * s + 1], oz = f.stencil[3 * s + 2];
                const int js = cell_probe(keys + hb, H, cx + ox, cy + oy, cz + oz);
                if (js < 0) continue;
                const int j0 = start[hb + js], jc = cnt[hb + js];
                // i relative to the neighbour cell's centre
                const float xs = ri.x - (float)ox * cellf, ys = ri.y - (float)oy * cellf,
                            zs = ri.z - (float)oz * cellf;
                for (int jb = 0; jb < jc; jb += 32) {
                    const int nt = min(32, jc - jb);
                    __syncwarp();
                    if (lane < nt) {
                        const size_t kj = nb + j0 + jb + lane;
                        T.rel[lane] = s_rel[kj];
                        T.pos[lane] = s_pos[kj];
                        T.par[lane] = s_par[kj];
                        T.aux[lane] = s_aux[kj];
                    }
                    __syncwarp();
                    if (!valid) continue;
                    unsigned mask = 0u;
                    for (int t = 0; t < nt; ++t) {
                        const float4 r = T.rel[t];
                        const float dx = xs - r.x, dy = ys - r.y, dz = zs - r.z;
                        const float d2 = dx * dx + dy * dy + dz * dz;
                        mask |= (d2 <= pre2 ? 1u : 0u) << t;
                    }
                    float fx = 0.f, fy = 0.f, fz = 0.f, fe = 0.f, fv = 0.f;
                    while (mask) {
                        const int t = __ffs(mask) - 1;
                        mask &= mask - 1u;
                        const int4 aj = T.aux[t];
                        const int j = aj.x;
                        if (j == i) continue;
                        const double4 pj = T.pos[t];
                        const double dx = xsub(pi4.x, pj.x), dy = xsub(pi4.y, pj.y), dz = xsub(pi4.z, pj.z);
                        const double d2 = d2_einsum(dx, dy, dz);
                        if (d2 > f.cut_pair2) continue;
                        const bool ke = d2 <= f.thr_elec2, kv = d2 <= f.thr_vdw2;
                        a.cnt += (int)ke + ((int)kv << 16);
                        double we, wv;
                        if (f.uniform_weights) {
                            we = wv = f.uniform_value;
                        } else {
                            int cls = 4;
                            if (ci && aj.z != 0 && abs(ai.y - aj.y) <= 1)
                                cls = classify_pair(f, i, j, pi, gpi, ggi, ai.y, true);
                            we = f.w_elec[cls - 1]; wv = f.w_vdw[cls - 1];
                        }
                        if (d2 < FP64_BELOW_D2) {
                            if (d2 < 1e-11) {
                                const double d = sqrt(d2);
                                if (d < MIN_DISTANCE) {
                                    atomicMin(&status[b].dmin_bits, (unsigned long long)__double_as_longlong(d));
                                    if (atomicCAS(&status[b].error, KF_ERR_NONE, KF_ERR_CLASH) == KF_ERR_NONE)
                                        status[b].err_iter = status[b].iter;
                                    continue;
                                }
                            }
                            pair_fp64(f, i, j, d2, dx, dy, dz, we, wv, ke, kv, a);
                            continue;
                        }
                        const float4 qj = T.par[t];
                        const float inv_r = rsqrtf((float)d2);
                        const float inv_r2 = inv_r * inv_r;
                        float g = 0.f;
                        if (ke) {
                            // kappa = d: E = K w qi qj / d^2, |F|/d = E / d^2;
                            // constant kappa: E = K w qi qj / (kappa d), |F|/d = E / d^2
                            const float qq = qi * qj.x * (float)we;
                            const float e = f.dielectric_const ? qq * kap_inv * inv_r : qq * inv_r2;
                            fe += e;
                            g += e * inv_r2;
                        }
                        if (kv) {
                            const float weps = (float)wv * qi4.z * qj.z;
                            const float D = qi4.y + qj.y;
                            const float sr = D * D * inv_r2;
                            const float s3 = sr * sr * sr;
                            const float s6 = s3 * s3;
                            fv += weps * (s6 - 2.f * s3);
                            g += 12.f * weps * (s6 - s3) * inv_r2;
                        }
                        fx += g * (float)dx; fy += g * (float)dy; fz += g * (float)dz;
                    }
                    a.fx += (double)fx; a.fy += (double)fy; a.fz += (double)fz;
                    a.ee += (double)fe; a.ev += (double)fv;
                }
            }
            if (valid) {
                const size_t o = nb + i;
                forces[3 * o] = a.fx; forces[3 * o + 1] = a.fy; forces[3 * o + 2] = a.fz;
                e_atom[2 * o] = a.ee; e_atom[2 * o + 1] = a.ev;
                pair_count[o] = a.cnt;
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
        g_pair_grid = sms * 8;
    }
    pair_kernel<<<g_pair_grid, PAIR_WARPS * 32, 0, s>>>(
        *f, w->B, n, w->cell_key, w->cell_cnt, w->cell_start, w->occ, w->occ_offset,
        reinterpret_cast<const float4 *>(w->s_rel), reinterpret_cast<const double4 *>(w->s_pos),
        reinterpret_cast<const float4 *>(w->s_par), reinterpret_cast<const int4 *>(w->s_aux), w->forces,
        w->e_atom, w->pair_count, w->status);
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
