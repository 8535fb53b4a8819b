// Nonbonded elec + vdW pair kernel (K3) with the cut-off filter (K2), the
// 1-2/1-3/1-4 classifier and the steric-clash guard fused in.
//
// Reference: Field.evaluate's force phase (/root/reference/pkg/src/kinefold/
// kcm.py:110-127) = extract_pairs (forcefield.py:81-89 -> spatial.py:233-241),
// TreeWeights.weights_for (topology.py:153-195), elec/vdw_pair_quantities
// (forcefield.py:98-113) and the bincount scatter (forcefield.py:162-172).
//
// Layout: one thread owns one atom (bucket order, so a warp covers a compact
// cluster) and walks the cell stencil; it computes every partner, both
// directions of each unordered pair are evaluated by their owners ("full list"),
// so forces need no atomics and the per-atom fp64 sums run in a fixed order:
// run-to-run bitwise deterministic.  Pair membership is decided exactly as the
// reference does (fp64 d2 in einsum order vs cut^2, and sqrt(d2) <= cut per
// term via the equivalent d2 thresholds); the pair energy/force math is fp32
// with fp64 per-atom accumulation, except pairs closer than 0.1 A which take
// the reference's fp64 formulas (fp32 (D/d)^12 overflows).
#include "kf_common.cuh"

namespace {

constexpr double COULOMB_K = 332.06;
constexpr double MIN_DISTANCE = 1e-6;
constexpr double FP64_BELOW_D2 = 1e-2;

KF_DEV void unpack_cell(long long p, int &cx, int &cy, int &cz) {
    const unsigned long long u = (unsigned long long)p;
    cx = (int)((long long)(u << 1) >> 43);
    cy = (int)((long long)(u << 22) >> 43);
    cz = (int)((long long)(u << 43) >> 43);
}

}  // namespace

namespace {

struct Acc {
    double fx, fy, fz, ee, ev;
    int cnt;
};

// Reference fp64 formulas for one pair (used at d < 0.1 A and by the API path).
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

__global__ void __launch_bounds__(128)
pair_kernel(kf_field_t f, int B, int n, const double *__restrict__ sorted_pos_d,
            const int32_t *__restrict__ sorted_atom, const int32_t *__restrict__ bstart,
            double *__restrict__ forces, double *__restrict__ e_atom, int32_t *__restrict__ pair_count,
            kf_status_t *status) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (long long)B * n) return;
    const int b = (int)(gid / n);
    if (status[b].done) return;
    const double4 *spos = reinterpret_cast<const double4 *>(sorted_pos_d) + (size_t)b * n;
    const int32_t *sid = sorted_atom + (size_t)b * n;
    const int H = 1 << f.hash_bits;
    const int32_t *st = bstart + (size_t)b * (H + 1);

    const int k = (int)(gid % n);
    const double4 me = spos[k];
    const int i = sid[k];
    int cx, cy, cz;
    unpack_cell(__double_as_longlong(me.w), cx, cy, cz);
    const float qi = f.q32[i] * (float)COULOMB_K, Ri = f.R32[i], si = f.seps32[i];
    int pi = -1, gpi = -1, ggi = -1, ri = 0;
    bool ci = false;
    if (!f.uniform_weights) {
        pi = f.tparent[i]; gpi = f.tgp[i]; ggi = f.tggp[i]; ri = f.tres[i]; ci = f.tchain[i] != 0;
    }
    const float kap_inv = f.dielectric_const ? (float)(1.0 / f.kappa) : 1.0f;
    Acc a = {0.0, 0.0, 0.0, 0.0, 0.0, 0};

    for (int s = 0; s < f.n_stencil; ++s) {
        const int ox = cx + f.stencil[3 * s], oy = cy + f.stencil[3 * s + 1], oz = cz + f.stencil[3 * s + 2];
        const long long key = pack_cell(ox, oy, oz);
        const uint32_t h = cell_hash(ox, oy, oz, (uint32_t)H - 1);
        const int s0 = st[h], s1 = st[h + 1];
        float fx = 0.f, fy = 0.f, fz = 0.f, ee = 0.f, ev = 0.f;
        for (int kk = s0; kk < s1; ++kk) {
            const double4 pj = spos[kk];
            if (__double_as_longlong(pj.w) != key || kk == k) continue;
            const double dx = xsub(me.x, pj.x), dy = xsub(me.y, pj.y), dz = xsub(me.z, pj.z);
            const double d2 = d2_einsum(dx, dy, dz);
            if (d2 > f.cut_pair2) continue;
            const int j = sid[kk];
            const bool ke = d2 <= f.thr_elec2, kv = d2 <= f.thr_vdw2;
            a.cnt += ke;
            double we, wv;
            if (f.uniform_weights) {
                we = wv = f.uniform_value;
            } else {
                const int cls = classify_pair(f, i, j, pi, gpi, ggi, ri, ci) - 1;
                we = f.w_elec[cls]; wv = f.w_vdw[cls];
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
            const float r2 = (float)d2;
            const float inv_r = rsqrtf(r2);
            const float inv_r2 = inv_r * inv_r;
            float g = 0.f;
            if (ke && we != 0.0) {
                // kappa = d: E = K w qi qj / d^2, |F|/d = E / d^2; constant kappa: E = K w qi qj /(kappa d)
                const float qq = qi * f.q32[j] * (float)we;
                const float e = f.dielectric_const ? qq * kap_inv * inv_r : qq * inv_r2;
                ee += e;
                g += e * inv_r2;
            }
            if (kv && wv != 0.0) {
                const float weps = (float)wv * si * f.seps32[j];
                const float D = Ri + f.R32[j];
                const float sr = D * D * inv_r2;
                const float s3 = sr * sr * sr;
                const float s6 = s3 * s3;
                ev += weps * (s6 - 2.f * s3);
                g += 12.f * weps * (s6 - s3) * inv_r2;
            }
            fx += g * (float)dx; fy += g * (float)dy; fz += g * (float)dz;
        }
        a.fx += (double)fx; a.fy += (double)fy; a.fz += (double)fz;
        a.ee += (double)ee; a.ev += (double)ev;
    }
    const size_t o = (size_t)b * n + i;
    forces[3 * o] = a.fx; forces[3 * o + 1] = a.fy; forces[3 * o + 2] = a.fz;
    e_atom[2 * o] = a.ee; e_atom[2 * o + 1] = a.ev;
    pair_count[o] = a.cnt;
}

// On error only: smallest (i, j), i < j, among pairs at the minimum distance.
__global__ void clash_report_kernel(kf_field_t f, int B, int n, const double *__restrict__ sorted_pos_d,
                                    const int32_t *__restrict__ sorted_atom,
                                    const int32_t *__restrict__ bstart, kf_status_t *status) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (long long)B * n) return;
    const int b = (int)(gid / n);
    if (status[b].error != KF_ERR_CLASH) return;
    const double4 *spos = reinterpret_cast<const double4 *>(sorted_pos_d) + (size_t)b * n;
    const int32_t *sid = sorted_atom + (size_t)b * n;
    const int H = 1 << f.hash_bits;
    const int32_t *st = bstart + (size_t)b * (H + 1);
    const int k = (int)(gid % n);
    const double4 me = spos[k];
    const int i = sid[k];
    int cx, cy, cz;
    unpack_cell(__double_as_longlong(me.w), cx, cy, cz);
    const unsigned long long target = status[b].dmin_bits;
    for (int s = 0; s < f.n_stencil; ++s) {
        const int ox = cx + f.stencil[3 * s], oy = cy + f.stencil[3 * s + 1], oz = cz + f.stencil[3 * s + 2];
        const long long key = pack_cell(ox, oy, oz);
        const uint32_t h = cell_hash(ox, oy, oz, (uint32_t)H - 1);
        for (int kk = st[h]; kk < st[h + 1]; ++kk) {
            const double4 pj = spos[kk];
            if (__double_as_longlong(pj.w) != key || kk == k) continue;
            const int j = sid[kk];
            if (j <= i) continue;
            const double d2 = d2_einsum(xsub(me.x, pj.x), xsub(me.y, pj.y), xsub(me.z, pj.z));
            if (d2 > f.cut_pair2) continue;
            if ((unsigned long long)__double_as_longlong(sqrt(d2)) == target) {
                const unsigned long long key_ij = ((unsigned long long)i << 32) | (unsigned)j;
                atomicMin(reinterpret_cast<unsigned long long *>(&status[b].clash_key), key_ij);
            }
        }
    }
}

}  // namespace

int kf_pairs_launch(const kf_field_t *f, kf_batch_t *w, int n, cudaStream_t s) {
    const long long total = (long long)w->B * n;
    pair_kernel<<<kf_blocks(total, 128), 128, 0, s>>>(*f, w->B, n, w->sorted_pos, w->sorted_atom,
                                                      w->bucket_start, w->forces, w->e_atom,
                                                      w->pair_count, w->status);
    KF_LAUNCH_CHECK("pair_kernel");
    return 0;
}

int kf_clash_report_launch(const kf_field_t *f, kf_batch_t *w, int n, cudaStream_t s) {
    const long long total = (long long)w->B * n;
    clash_report_kernel<<<kf_blocks(total, 128), 128, 0, s>>>(*f, w->B, n, w->sorted_pos, w->sorted_atom,
                                                              w->bucket_start, w->status);
    KF_LAUNCH_CHECK("clash_report_kernel");
    return 0;
}
