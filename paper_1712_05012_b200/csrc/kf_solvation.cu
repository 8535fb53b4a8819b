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
#include "kf_common.cuh"

namespace {

constexpr int SOLV_THREADS = 256;

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

// Shared body: states + (optionally) events for atom i against nn staged slots.
// Returns the number of covered samples.
template <bool WITH_FORCES>
KF_DEV int enumerate_samples(const double *xi, double r_off_i, const double *samples, int N,
                             const NbSlot *nb, int nn, long long wi, double dr, long long *acc_nb,
                             long long *acc_i, uint8_t *counts_out, int32_t *crit_out,
                             const int32_t *nb_atom) {
    int covered = 0;
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        double px, py, pz;
        sample_point(xi, r_off_i, samples + 3 * k, px, py, pz);
        int cnt = 0, crit = -1;
        for (int m = 0; m < nn; ++m) {
            if (covers(px, py, pz, nb[m])) {
                crit = m;
                if (++cnt == 2) break;
            }
        }
        covered += cnt > 0;
        if (counts_out) {
            counts_out[k] = (uint8_t)cnt;
            crit_out[k] = cnt == 1 ? nb_atom[crit] : -1;
        }
        if (WITH_FORCES && wi != 0) {
            if (cnt == 0) {
                for (int s = 0; s < 3; ++s) {
                    for (int m = 0; m < nn; ++m) {
                        if (covers_shifted(px, py, pz, nb[m], s, dr)) {
                            atomicAdd(reinterpret_cast<unsigned long long *>(&acc_nb[3 * m + s]),
                                      (unsigned long long)wi);
                            acc_i[s] -= wi;
                        }
                    }
                }
            } else if (cnt == 1) {
                for (int s = 0; s < 3; ++s) {
                    if (!covers_shifted(px, py, pz, nb[crit], s, dr)) {
                        acc_i[s] += wi;
                        atomicAdd(reinterpret_cast<unsigned long long *>(&acc_nb[3 * crit + s]),
                                  (unsigned long long)(-wi));
                    }
                }
            }
        }
    }
    return covered;
}

// Hot path: neighbours come from the spatial hash of this iteration.
__global__ void __launch_bounds__(SOLV_THREADS)
solv_hot_kernel(kf_field_t f, int n, int n_solv, const int32_t *__restrict__ solv_atoms,
                const double *__restrict__ pos_all, const unsigned long long *__restrict__ keys,
                const int32_t *__restrict__ cnt, const int32_t *__restrict__ start,
                const int32_t *__restrict__ atom_slot, const double4 *__restrict__ s_pos,
                const int4 *__restrict__ s_aux, long long *__restrict__ solv_acc,
                double *__restrict__ cav_atom, double *__restrict__ f_exp_out,
                double *__restrict__ a_exp_out, int nb_cap, kf_status_t *status) {
    const int b = blockIdx.x / n_solv;
    const int i = solv_atoms[blockIdx.x % n_solv];
    if (status[b].done) return;
    extern __shared__ __align__(16) unsigned char smem[];
    NbSlot *nb = reinterpret_cast<NbSlot *>(smem);
    long long *acc_nb = reinterpret_cast<long long *>(nb + nb_cap);
    int32_t *nb_atom = reinterpret_cast<int32_t *>(acc_nb + 3 * nb_cap);
    __shared__ int nn;
    __shared__ long long acc_i_s[3];
    __shared__ double red[32];
    if (threadIdx.x == 0) { nn = 0; acc_i_s[0] = acc_i_s[1] = acc_i_s[2] = 0; }
    __syncthreads();

    const size_t ai = (size_t)b * n + i;
    const double xi[3] = {pos_all[3 * ai], pos_all[3 * ai + 1], pos_all[3 * ai + 2]};
    const double r_off_i = f.r_off[i];
    const uint32_t H = 1u << f.hash_bits;
    const size_t hb = (size_t)b * H, nbase = (size_t)b * n;
    int cx, cy, cz;
    unpack_cell((long long)keys[hb + atom_slot[ai]], cx, cy, cz);

    for (int s = threadIdx.x; s < f.n_stencil; s += blockDim.x) {
        const int js = cell_probe(keys + hb, H, cx + f.stencil[3 * s], cy + f.stencil[3 * s + 1],
                                  cz + f.stencil[3 * s + 2]);
        if (js < 0) continue;
        for (int kk = start[hb + js]; kk < start[hb + js] + cnt[hb + js]; ++kk) {
            const double4 pj = s_pos[nbase + kk];
            const int j = s_aux[nbase + kk].x;
            if (j == i) continue;
            const double dx = xi[0] - pj.x, dy = xi[1] - pj.y, dz = xi[2] - pj.z;
            const double lim = r_off_i + f.r_off[j] + f.reach_pad;
            if (dx * dx + dy * dy + dz * dz > lim * lim) continue;
            const int slot = atomicAdd(&nn, 1);
            if (slot < nb_cap) {
                nb[slot] = NbSlot{pj.x, pj.y, pj.z, f.r_off2[j]};
                nb_atom[slot] = j;
            }
        }
    }
    __syncthreads();
    const int count = nn;
    if (count > nb_cap) {
        if (threadIdx.x == 0) {
            atomicMax(&status[b].overflow, count);
            if (atomicCAS(&status[b].error, KF_ERR_NONE, KF_ERR_CAPACITY) == KF_ERR_NONE)
                status[b].err_iter = status[b].iter;
        }
        return;
    }
    for (int m = threadIdx.x; m < 3 * count; m += blockDim.x) acc_nb[m] = 0;
    __syncthreads();

    long long acc_i[3] = {0, 0, 0};
    const long long wi = f.w_int[i];
    const int covered = enumerate_samples<true>(xi, r_off_i, f.samples, f.n_samples, nb, count, wi,
                                                f.delta_r, acc_nb, acc_i, nullptr, nullptr, nb_atom);
    const double cov_total = block_sum((double)covered, red);
    for (int s = 0; s < 3; ++s) {
        const long long v = warp_sum_ll(acc_i[s]);
        if ((threadIdx.x & 31) == 0 && v != 0)
            atomicAdd(reinterpret_cast<unsigned long long *>(&acc_i_s[s]), (unsigned long long)v);
    }
    __syncthreads();
    long long *acc = solv_acc + (size_t)b * n * 3;
    for (int m = threadIdx.x; m < 3 * count; m += blockDim.x) {
        const long long v = acc_nb[m];
        if (v != 0)
            atomicAdd(reinterpret_cast<unsigned long long *>(&acc[3 * (size_t)nb_atom[m / 3] + m % 3]),
                      (unsigned long long)v);
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < 3; ++s)
            if (acc_i_s[s] != 0)
                atomicAdd(reinterpret_cast<unsigned long long *>(&acc[3 * (size_t)i + s]),
                          (unsigned long long)acc_i_s[s]);
        // f_exp = (N - covered) / N; a_exp = f_exp * (4 pi R_off^2); term = gamma * a_exp
        const long long cov = (long long)cov_total;
        const double f_exp = (double)(f.n_samples - cov) / (double)f.n_samples;
        const double a_exp = xmul(f_exp, xmul(f.four_pi, f.r_off2[i]));
        cav_atom[ai] = xmul(f.gamma[i], a_exp);
        if (f_exp_out) { f_exp_out[ai] = f_exp; a_exp_out[ai] = a_exp; }
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
    NbSlot *nb = reinterpret_cast<NbSlot *>(smem);
    int32_t *nb_atom = reinterpret_cast<int32_t *>(nb + nb_cap);
    __shared__ int nn;
    __shared__ double red[32];
    if (threadIdx.x == 0) nn = 0;
    __syncthreads();
    const int count = stage_from_list(pos, r_off, r_off2, i, nb_off, nbl, pad, nb, nb_atom, nb_cap, &nn);
    if (count > nb_cap) {
        if (threadIdx.x == 0) atomicMax(overflow, count);
        return;
    }
    const double xi[3] = {pos[3 * (size_t)i], pos[3 * (size_t)i + 1], pos[3 * (size_t)i + 2]};
    const bool empty_list = nb_off[i + 1] == nb_off[i];
    const int cov = enumerate_samples<false>(xi, r_off[i], samples, N, nb, count, 0, 0.0, nullptr,
                                             nullptr, counts + (size_t)i * N, critical + (size_t)i * N,
                                             nb_atom);
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
    NbSlot *nb = reinterpret_cast<NbSlot *>(smem);
    long long *acc_nb = reinterpret_cast<long long *>(nb + nb_cap);
    int32_t *nb_atom = reinterpret_cast<int32_t *>(acc_nb + 3 * nb_cap);
    __shared__ int nn;
    __shared__ long long acc_i_s[3];
    if (threadIdx.x == 0) { nn = 0; acc_i_s[0] = acc_i_s[1] = acc_i_s[2] = 0; }
    __syncthreads();
    const int count = stage_from_list(pos, r_off, r_off2, i, nb_off, nbl, pad, nb, nb_atom, nb_cap, &nn);
    if (count > nb_cap) {
        if (threadIdx.x == 0) atomicMax(overflow, count);
        return;
    }
    for (int m = threadIdx.x; m < 3 * count; m += blockDim.x) acc_nb[m] = 0;
    __syncthreads();
    const double xi[3] = {pos[3 * (size_t)i], pos[3 * (size_t)i + 1], pos[3 * (size_t)i + 2]};
    long long acc_i[3] = {0, 0, 0};
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        const int c = counts[(size_t)i * N + k];
        if (c > 1) continue;
        double px, py, pz;
        sample_point(xi, r_off[i], samples + 3 * k, px, py, pz);
        if (c == 0) {
            for (int s = 0; s < 3; ++s)
                for (int m = 0; m < count; ++m)
                    if (covers_shifted(px, py, pz, nb[m], s, dr)) {
                        atomicAdd(reinterpret_cast<unsigned long long *>(&acc_nb[3 * m + s]),
                                  (unsigned long long)wi);
                        acc_i[s] -= wi;
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

size_t hot_smem(int cap) { return (size_t)cap * (sizeof(NbSlot) + 3 * sizeof(long long) + sizeof(int32_t)); }

}  // namespace

int kf_solvation_launch(const kf_field_t *f, kf_batch_t *w, int n, int n_solv, const int32_t *solv_atoms,
                        cudaStream_t s) {
    const int B = w->B;
    KF_CUDA(cudaMemsetAsync(w->solv_acc, 0, sizeof(long long) * (size_t)B * n * 3, s), "memset solv_acc");
    if (n_solv > 0) {
        const size_t smem = hot_smem(w->nb_cap);
        static size_t opted = 0;
        if (smem > 48 * 1024 && smem > opted) {
            KF_CUDA(cudaFuncSetAttribute(solv_hot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                    "smem attr");
            opted = smem;
        }
        solv_hot_kernel<<<(unsigned)((long long)B * n_solv), SOLV_THREADS, smem, s>>>(
            *f, n, n_solv, solv_atoms, w->pos, w->cell_key, w->cell_cnt, w->cell_start, w->atom_slot,
            reinterpret_cast<const double4 *>(w->s_pos), reinterpret_cast<const int4 *>(w->s_aux), w->solv_acc, w->cav_atom, w->f_exp, w->a_exp, w->nb_cap, w->status);
        KF_LAUNCH_CHECK("solv_hot_kernel");
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
    const size_t smem = (size_t)nb_cap * (sizeof(NbSlot) + sizeof(int32_t));
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
    const size_t smem = hot_smem(nb_cap);
    if (smem > 48 * 1024)
        KF_CUDA(cudaFuncSetAttribute(solv_forces_api_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem), "smem attr");
    solv_forces_api_kernel<<<n, SOLV_THREADS, smem, s>>>(pos, r_off, r_off2, w_int, samples, N, nb_off, nb,
                                                          counts, critical, dr, pad, acc, nb_cap, overflow);
    KF_LAUNCH_CHECK("solv_forces_api_kernel");
    return 0;
}
