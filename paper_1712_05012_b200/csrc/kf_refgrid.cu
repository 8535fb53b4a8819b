// Reference-API spatial kernels: the bit-exact reference grid (build_grid),
// the superset neighbour table (build_neighbor_table), table filtering
// (filtered_pairs / filtered_lists / extract_pairs), pair classification and
// the table-driven elec/vdW terms of the forcefield API functions.
//
// Reference: /root/reference/pkg/src/kinefold/spatial.py:83-259,
// topology.py:153-195, forcefield.py:81-172.  These serve the drop-in API
// calls and the parity tests; the KCM loop itself uses the fused hash-grid
// kernels (kf_grid.cu, kf_nonbonded.cu).
#include "kf_common.cuh"


namespace {

// ---- generic scans / sums ------------------------------------------------------
constexpr int SCAN_T = 1024;

// exclusive scan of in[0..n) into out[0..n] (out[n] = total) for one block's range
__global__ void __launch_bounds__(SCAN_T)
scan_blocks_kernel(const int64_t *__restrict__ in, int64_t n, int64_t per_block, int64_t *__restrict__ out,
                   int64_t *__restrict__ block_sums) {
    const int64_t base = (int64_t)blockIdx.x * per_block;
    const int64_t end = min(n, base + per_block);
    const int64_t per = (per_block + SCAN_T - 1) / SCAN_T;
    const int64_t lo = min(end, base + (int64_t)threadIdx.x * per), hi = min(end, lo + per);
    long long local = 0;
    for (int64_t k = lo; k < hi; ++k) local += in[k];
    __shared__ long long ws[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long incl = local;
    for (int o = 1; o < 32; o <<= 1) {
        long long v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) ws[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        long long v = ws[lane];
        for (int o = 1; o < 32; o <<= 1) {
            long long u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        ws[lane] = v;
    }
    __syncthreads();
    long long run = incl - local + (wid > 0 ? ws[wid - 1] : 0);
    for (int64_t k = lo; k < hi; ++k) { out[k] = run; run += in[k]; }
    if (threadIdx.x == SCAN_T - 1) block_sums[blockIdx.x] = run;
}

__global__ void scan_fixup_kernel(int64_t n, int64_t per_block, const int64_t *__restrict__ block_sums,
                                  int nblocks, int64_t *__restrict__ out) {
    // block_sums scanned serially by thread 0 of each block (nblocks is small)
    __shared__ long long offset;
    if (threadIdx.x == 0) {
        long long acc = 0;
        for (int k = 0; k < (int)blockIdx.x; ++k) acc += block_sums[k];
        offset = acc;
        if (blockIdx.x == (unsigned)nblocks - 1) {
            long long tot = acc + block_sums[blockIdx.x];
            out[n] = tot;
        }
    }
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * per_block;
    const int64_t end = min(n, base + per_block);
    for (int64_t k = base + threadIdx.x; k < end; k += blockDim.x) out[k] += offset;
}

__global__ void i32_to_i64_kernel(const int32_t *in, int64_t n, int64_t *out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) out[k] = in[k];
}

__global__ void u8_to_i64_kernel(const uint8_t *in, int64_t n, int64_t *out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) out[k] = in[k];
}

// deterministic fp64 sum: fixed chunking, fixed tree
__global__ void __launch_bounds__(1024) sum_partials_kernel(const double *x, int64_t n, int64_t per_block,
                                                            double *partials) {
    __shared__ double red[32];
    const int64_t base = (int64_t)blockIdx.x * per_block, end = min(n, base + per_block);
    double s = 0.0;
    for (int64_t k = base + threadIdx.x; k < end; k += blockDim.x) s += x[k];
    s = block_sum(s, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}
__global__ void __launch_bounds__(1024) sum_final_kernel(const double *partials, int nb, double *out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int k = threadIdx.x; k < nb; k += blockDim.x) s += partials[k];
    s = block_sum(s, red);
    if (threadIdx.x == 0) *out = s;
}

// ---- build_grid ------------------------------------------------------------------
__global__ void __launch_bounds__(1024) bbox_kernel(const double *pos, int n, double *out) {
    __shared__ double red[32];
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    double bad = 0.0;
    for (int a = threadIdx.x; a < n; a += blockDim.x)
        for (int k = 0; k < 3; ++k) {
            const double v = pos[3 * (size_t)a + k];
            if (!isfinite(v)) bad += 1.0;
            mn[k] = fmin(mn[k], v);
            mx[k] = fmax(mx[k], v);
        }
    for (int k = 0; k < 3; ++k) {
        const double lo = -block_max(-mn[k], red);
        const double hi = block_max(mx[k], red);
        if (threadIdx.x == 0) { out[k] = lo; out[3 + k] = hi; }
    }
    bad = block_sum(bad, red);
    if (threadIdx.x == 0) out[6] = bad;
}

// cells = clip(floor((r - r_min) / cell), 0, dims - 1); lin = (c0 d1 + c1) d2 + c2
// (spatial.py:97-99): one IEEE subtract and one IEEE divide per component.
__global__ void grid_cells_kernel(const double *pos, int n, const double *r_min, double cell,
                                  const int64_t *dims, int64_t *cell_index, int64_t *lin) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    int64_t c[3];
    for (int k = 0; k < 3; ++k) {
        const double q = __ddiv_rn(xsub(pos[3 * (size_t)a + k], r_min[k]), cell);
        int64_t v = (int64_t)floor(q);
        v = v < 0 ? 0 : (v > dims[k] - 1 ? dims[k] - 1 : v);
        c[k] = v;
        cell_index[3 * (size_t)a + k] = v;
    }
    lin[a] = (c[0] * dims[1] + c[1]) * dims[2] + c[2];
}

__global__ void count_keys_kernel(const int64_t *key, int n, int32_t *counts) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a < n) atomicAdd(&counts[key[a]], 1);
}
__global__ void scatter_keys_kernel(const int64_t *key, int n, const int64_t *starts, int32_t *cursor,
                                    int64_t *order) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a < n) order[starts[key[a]] + atomicAdd(&cursor[key[a]], 1)] = a;
}
// insertion sort of each key's members (stable order = ascending atom index)
__global__ void sort_segments_kernel(const int64_t *starts, int64_t n_seg, int64_t *vals) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    const int64_t lo = starts[s], hi = starts[s + 1];
    for (int64_t k = lo + 1; k < hi; ++k) {
        const int64_t v = vals[k];
        int64_t m = k - 1;
        while (m >= lo && vals[m] > v) { vals[m + 1] = vals[m]; --m; }
        vals[m + 1] = v;
    }
}

// ---- build_neighbor_table -----------------------------------------------------------
KF_DEV bool stencil_cell(const int64_t *ci, const int64_t *dims, const int32_t *off, int64_t &lin) {
    int64_t c[3];
    for (int k = 0; k < 3; ++k) {
        c[k] = ci[k] + off[k];
        if (c[k] < 0 || c[k] >= dims[k]) return false;
    }
    lin = (c[0] * dims[1] + c[1]) * dims[2] + c[2];
    return true;
}

__global__ void rows_count_kernel(const int64_t *cell_index, const int64_t *dims, int n,
                                  const int64_t *cell_start, const int32_t *stencil, int n_stencil,
                                  int64_t *row_len) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    int64_t total = 0, lin;
    for (int s = 0; s < n_stencil; ++s)
        if (stencil_cell(cell_index + 3 * (size_t)a, dims, stencil + 3 * s, lin))
            total += cell_start[lin + 1] - cell_start[lin];
    row_len[a] = total - 1;   // self excluded
}

__global__ void rows_fill_kernel(const int64_t *cell_index, const int64_t *dims, int n,
                                 const int64_t *cell_start, const int64_t *order, const int32_t *stencil,
                                 int n_stencil, const int64_t *offsets, int64_t *neighbors) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    int64_t w = offsets[a], lin;
    for (int s = 0; s < n_stencil; ++s)
        if (stencil_cell(cell_index + 3 * (size_t)a, dims, stencil + 3 * s, lin))
            for (int64_t e = cell_start[lin]; e < cell_start[lin + 1]; ++e)
                if (order[e] != a) neighbors[w++] = order[e];
}

constexpr int ROWSORT_MAX = 8192;

// one CTA per row: bitonic sort in shared memory; longer rows: serial insertion
__global__ void __launch_bounds__(1024) sort_rows_kernel(const int64_t *offsets, int64_t *vals) {
    extern __shared__ long long buf[];
    const int64_t lo = offsets[blockIdx.x], hi = offsets[blockIdx.x + 1];
    const int len = (int)(hi - lo);
    if (len < 2) return;
    if (len > ROWSORT_MAX) {
        if (threadIdx.x == 0)
            for (int64_t k = lo + 1; k < hi; ++k) {
                const int64_t v = vals[k];
                int64_t m = k - 1;
                while (m >= lo && vals[m] > v) { vals[m + 1] = vals[m]; --m; }
                vals[m + 1] = v;
            }
        return;
    }
    int p2 = 1;
    while (p2 < len) p2 <<= 1;
    for (int k = threadIdx.x; k < p2; k += blockDim.x) buf[k] = k < len ? vals[lo + k] : LLONG_MAX;
    __syncthreads();
    for (int size = 2; size <= p2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < p2; t += blockDim.x) {
                const int partner = t ^ stride;
                if (partner > t) {
                    const bool up = (t & size) == 0;
                    const long long x = buf[t], y = buf[partner];
                    if ((x > y) == up) { buf[t] = y; buf[partner] = x; }
                }
            }
            __syncthreads();
        }
    for (int k = threadIdx.x; k < len; k += blockDim.x) vals[lo + k] = buf[k];
}

// ---- filtered_pairs / filtered_lists ---------------------------------------------
__global__ void filter_table_kernel(const double *pos, const int64_t *offsets, const int64_t *neighbors,
                                    int n, int64_t n_entries, double cut2, int upper_only, uint8_t *keep,
                                    double *d2_out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_entries) return;
    int lo = 0, hi = n;   // row = largest r with offsets[r] <= e
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (offsets[mid] <= e) lo = mid; else hi = mid;
    }
    const int i = lo;
    const int64_t j = neighbors[e];
    if (upper_only && j <= i) { keep[e] = 0; return; }
    const double *a = pos + 3 * (size_t)i, *b = pos + 3 * (size_t)j;
    const double d2 = d2_einsum(xsub(a[0], b[0]), xsub(a[1], b[1]), xsub(a[2], b[2]));
    d2_out[e] = d2;
    keep[e] = d2 <= cut2;
}

__global__ void compact_pairs_kernel(const int64_t *offsets, const int64_t *neighbors, int n,
                                     int64_t n_entries, const uint8_t *keep, const int64_t *dest,
                                     const double *d2, int64_t *oi, int64_t *oj, double *od) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_entries || !keep[e]) return;
    int lo = 0, hi = n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (offsets[mid] <= e) lo = mid; else hi = mid;
    }
    const int64_t k = dest[e];
    if (oi) oi[k] = lo;
    oj[k] = neighbors[e];
    if (od) od[k] = sqrt(d2[e]);
}

// ---- classification + table-driven pair terms -----------------------------------
__global__ void classify_kernel(kf_field_t f, const int64_t *pi_, const int64_t *pj_, int64_t m,
                                int64_t *cls) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= m) return;
    const int i = (int)pi_[p], j = (int)pj_[p];
    cls[p] = classify_pair(f, i, j, f.tparent[i], f.tgp[i], f.tggp[i], f.tres[i], f.tchain[i] != 0);
}

// Reference formulas verbatim in fp64 (forcefield.py:98-113, :162-172).
__global__ void pair_terms_kernel(kf_field_t f, const double *pos, const int64_t *pi_, const int64_t *pj_,
                                  const double *dd_, const double *w_in, int64_t m, int kind, double *e_out,
                                  double *mag_out, double *fvec) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= m) return;
    const int i = (int)pi_[p], j = (int)pj_[p];
    const double d = dd_[p];
    double w;
    if (w_in) {
        w = w_in[p];
    } else if (f.uniform_weights) {
        w = f.uniform_value;
    } else {
        const int cls = classify_pair(f, i, j, f.tparent[i], f.tgp[i], f.tggp[i], f.tres[i], f.tchain[i] != 0);
        w = kind == 0 ? f.w_elec[cls - 1] : f.w_vdw[cls - 1];
    }
    double e, mag;
    if (kind == 0) {
        const double kap = f.dielectric_const ? f.kappa : d;
        const double num = 332.06 * w * f.q[i] * f.q[j];
        e = num / (kap * d);
        mag = num / (kap * d * d);
    } else {
        const double eps = sqrt(f.eps[i] * f.eps[j]);
        const double dd = f.R[i] + f.R[j];
        const double ratio6 = pow(dd, 6.0) / pow(d, 6.0);
        e = w * eps * (ratio6 * ratio6 - 2.0 * ratio6);
        mag = 12.0 * w * eps * (pow(dd, 12.0) / pow(d, 13.0) - pow(dd, 6.0) / pow(d, 7.0));
    }
    if (e_out) e_out[p] = e;
    if (mag_out) mag_out[p] = mag;
    if (fvec)   // e = (r_i - r_j) / d; f = mag e (forcefield.py:167-168); scattered by bincount_apply
        for (int k = 0; k < 3; ++k)
            fvec[3 * p + k] = mag * ((pos[3 * (size_t)i + k] - pos[3 * (size_t)j + k]) / d);
}

// Per-pair force vectors f = mag * ((r_i - r_j) / d) (forcefield.py:167-168).
__global__ void pair_fvec_kernel(const double *pos, const int64_t *pi_, const int64_t *pj_, const double *dd_,
                                 const double *mag, int64_t m, double *fvec) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= m) return;
    const int64_t i = pi_[p], j = pj_[p];
    for (int k = 0; k < 3; ++k) fvec[3 * p + k] = mag[p] * ((pos[3 * i + k] - pos[3 * j + k]) / dd_[p]);
}

// The reference's scatter, bit for bit (forcefield.py:169-171): per component,
// out += np.bincount(i, f), then out -= np.bincount(j, f).  np.bincount adds
// the weights of each bin sequentially in pair order starting from 0.0; the
// stable counting sorts by i and by j list each atom's pairs in that order, so
// one thread per atom reproduces both sums and the result is deterministic.
__global__ void bincount_apply_kernel(int n, const int64_t *st_i, const int64_t *ord_i, const int64_t *st_j,
                                      const int64_t *ord_j, const double *fvec, double *forces) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    for (int k = 0; k < 3; ++k) {
        double si = 0.0, sj = 0.0;
        for (int64_t e = st_i[a]; e < st_i[a + 1]; ++e) si = xadd(si, fvec[3 * ord_i[e] + k]);
        for (int64_t e = st_j[a]; e < st_j[a + 1]; ++e) sj = xadd(sj, fvec[3 * ord_j[e] + k]);
        forces[3 * (size_t)a + k] = xsub(xadd(forces[3 * (size_t)a + k], si), sj);
    }
}

__global__ void occupied_kernel(const int32_t *counts, const int64_t *starts, const int64_t *dest, int64_t n_keys,
                                int64_t *occupied, int64_t *occ_starts) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_keys || counts[k] == 0) return;
    occupied[dest[k]] = k;
    occ_starts[dest[k]] = starts[k];
}
__global__ void nonzero_flags_kernel(const int32_t *counts, int64_t n, int64_t *flags) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) flags[k] = counts[k] != 0;
}
__global__ void row_kept_kernel(const int64_t *offsets, int n, const int64_t *dest, int64_t *out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r <= n) out[r] = dest[offsets[r]];
}
__global__ void argmin_kernel(const double *x, int64_t m, int64_t *out) {
    // smallest value, first index among equals (np.argmin)
    __shared__ double bv[1024];
    __shared__ int64_t bi[1024];
    double v = INFINITY;
    int64_t idx = -1;
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x)
        if (x[k] < v || (x[k] == v && (idx < 0 || k < idx))) { v = x[k]; idx = k; }
    bv[threadIdx.x] = v; bi[threadIdx.x] = idx;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) {
            const double v2 = bv[threadIdx.x + s];
            const int64_t i2 = bi[threadIdx.x + s];
            if (i2 >= 0 && (v2 < bv[threadIdx.x] || (v2 == bv[threadIdx.x] && (bi[threadIdx.x] < 0 || i2 < bi[threadIdx.x])))) {
                bv[threadIdx.x] = v2; bi[threadIdx.x] = i2;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = bi[0];
}

}  // namespace

// ---- host wrappers ------------------------------------------------------------------
int kf_scan_i64(const int64_t *in, int64_t n, int64_t *out, int64_t *scratch, cudaStream_t s) {
    // out[0..n] exclusive; scratch >= 1024 entries
    if (n == 0) {
        KF_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s), "scan memset");
        return 0;
    }
    int64_t per_block = 1 << 16;
    int nb = (int)((n + per_block - 1) / per_block);
    while (nb > 1024) { per_block <<= 1; nb = (int)((n + per_block - 1) / per_block); }
    scan_blocks_kernel<<<nb, SCAN_T, 0, s>>>(in, n, per_block, out, scratch);
    KF_LAUNCH_CHECK("scan_blocks_kernel");
    scan_fixup_kernel<<<nb, 256, 0, s>>>(n, per_block, scratch, nb, out);
    KF_LAUNCH_CHECK("scan_fixup_kernel");
    return 0;
}

int kf_sum_f64_launch(const double *x, int64_t n, double *partials /* >= 1024 */, double *out, cudaStream_t s) {
    int64_t per_block = 1 << 14;
    int nb = (int)((n + per_block - 1) / per_block);
    if (nb < 1) nb = 1;
    while (nb > 1024) { per_block <<= 1; nb = (int)((n + per_block - 1) / per_block); }
    sum_partials_kernel<<<nb, 1024, 0, s>>>(x, n, per_block, partials);
    KF_LAUNCH_CHECK("sum_partials_kernel");
    sum_final_kernel<<<1, 1024, 0, s>>>(partials, nb, out);
    KF_LAUNCH_CHECK("sum_final_kernel");
    return 0;
}

int kf_u8_to_i64_launch(const uint8_t *in, int64_t n, int64_t *out, cudaStream_t s) {
    if (n == 0) return 0;
    u8_to_i64_kernel<<<kf_blocks(n, 256), 256, 0, s>>>(in, n, out);
    KF_LAUNCH_CHECK("u8_to_i64_kernel");
    return 0;
}

int kf_counting_sort_launch(const int64_t *key, int n, int64_t n_keys, int32_t *counts, int64_t *starts,
                            int64_t *order, int64_t *scratch, cudaStream_t s);

// forces[a] = (forces[a] + bincount(i, f)[a]) - bincount(j, f)[a] for the m
// per-pair vectors fvec (stream-ordered scratch for the two stable sorts).
static int scatter_bincount(int n, const int64_t *i, const int64_t *j, int64_t m, const double *fvec,
                            double *forces, cudaStream_t s) {
    if (m > 0x7fffffffLL) { kf_set_error("scatter_bincount", cudaErrorInvalidValue); return 1; }
    const size_t bytes = sizeof(int32_t) * (size_t)n + sizeof(int64_t) * (2 * ((size_t)n + 1) + 2 * (size_t)m +
                                                                          (size_t)n + 1024);
    char *buf = nullptr;
    KF_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&buf), bytes, s), "scatter scratch");
    int64_t *st_i = reinterpret_cast<int64_t *>(buf), *st_j = st_i + n + 1, *ord_i = st_j + n + 1,
            *ord_j = ord_i + m, *scratch = ord_j + m;
    int32_t *counts = reinterpret_cast<int32_t *>(scratch + n + 1024);
    int rc = kf_counting_sort_launch(i, (int)m, n, counts, st_i, ord_i, scratch, s);
    if (!rc) rc = kf_counting_sort_launch(j, (int)m, n, counts, st_j, ord_j, scratch, s);
    if (!rc && n > 0) {
        bincount_apply_kernel<<<kf_blocks(n, 128), 128, 0, s>>>(n, st_i, ord_i, st_j, ord_j, fvec, forces);
        kf_count_launch();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { kf_set_error("bincount_apply_kernel", e); rc = 1; }
    }
    cudaError_t e = cudaFreeAsync(buf, s);
    if (!rc && e != cudaSuccess) { kf_set_error("scatter scratch free", e); rc = 1; }
    return rc;
}

extern "C" {

int kf_bbox(const double *pos, int n, double *out, void *stream) {
    bbox_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(pos, n, out);
    KF_LAUNCH_CHECK("bbox_kernel");
    return 0;
}

int kf_grid_cells(const double *pos, int n, const double *r_min, double cell, const int64_t *dims,
                  int64_t *cell_index, int64_t *lin, void *stream) {
    if (n == 0) return 0;
    grid_cells_kernel<<<kf_blocks(n, 256), 256, 0, (cudaStream_t)stream>>>(pos, n, r_min, cell, dims, cell_index, lin);
    KF_LAUNCH_CHECK("grid_cells_kernel");
    return 0;
}

int kf_counting_sort(const int64_t *key, int n, int64_t n_keys, int32_t *counts, int64_t *starts,
                     int64_t *order, int64_t *scratch, void *stream) {
    return kf_counting_sort_launch(key, n, n_keys, counts, starts, order, scratch, (cudaStream_t)stream);
}

}  // extern "C"

int kf_counting_sort_launch(const int64_t *key, int n, int64_t n_keys, int32_t *counts, int64_t *starts,
                            int64_t *order, int64_t *scratch, cudaStream_t s) {
    KF_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * n_keys, s), "memset counts");
    if (n > 0) {
        count_keys_kernel<<<kf_blocks(n, 256), 256, 0, s>>>(key, n, counts);
        KF_LAUNCH_CHECK("count_keys_kernel");
    }
    // widen counts into scratch[0..n_keys), scan into starts (block sums after them)
    int64_t *wide = scratch;
    i32_to_i64_kernel<<<kf_blocks(n_keys, 256), 256, 0, s>>>(counts, n_keys, wide);
    KF_LAUNCH_CHECK("i32_to_i64_kernel");
    if (kf_scan_i64(wide, n_keys, starts, scratch + n_keys, s)) return 1;
    KF_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * n_keys, s), "memset cursor");
    if (n > 0) {
        scatter_keys_kernel<<<kf_blocks(n, 256), 256, 0, s>>>(key, n, starts, counts, order);
        KF_LAUNCH_CHECK("scatter_keys_kernel");
        sort_segments_kernel<<<kf_blocks(n_keys, 256), 256, 0, s>>>(starts, n_keys, order);
        KF_LAUNCH_CHECK("sort_segments_kernel");
    }
    return 0;
}

extern "C" {

int kf_neighbor_rows_count(const int64_t *cell_index, const int64_t *dims, int n, const int64_t *cell_start,
                           const int32_t *stencil, int n_stencil, int64_t *row_len, void *stream) {
    if (n == 0) return 0;
    rows_count_kernel<<<kf_blocks(n, 128), 128, 0, (cudaStream_t)stream>>>(cell_index, dims, n, cell_start,
                                                                           stencil, n_stencil, row_len);
    KF_LAUNCH_CHECK("rows_count_kernel");
    return 0;
}

int kf_neighbor_rows_fill(const int64_t *cell_index, const int64_t *dims, int n, const int64_t *cell_start,
                          const int64_t *order, const int32_t *stencil, int n_stencil, const int64_t *offsets,
                          int64_t *neighbors, void *stream) {
    if (n == 0) return 0;
    rows_fill_kernel<<<kf_blocks(n, 128), 128, 0, (cudaStream_t)stream>>>(cell_index, dims, n, cell_start, order,
                                                                          stencil, n_stencil, offsets, neighbors);
    KF_LAUNCH_CHECK("rows_fill_kernel");
    return 0;
}

int kf_sort_rows(const int64_t *offsets, int n_rows, int64_t *values, void *stream) {
    if (n_rows == 0) return 0;
    static bool opted = false;
    const int smem = ROWSORT_MAX * (int)sizeof(long long);
    if (!opted) {
        KF_CUDA(cudaFuncSetAttribute(sort_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                "sort_rows smem");
        opted = true;
    }
    sort_rows_kernel<<<n_rows, 1024, smem, (cudaStream_t)stream>>>(offsets, values);
    KF_LAUNCH_CHECK("sort_rows_kernel");
    return 0;
}

int kf_filter_table(const double *pos, const int64_t *offsets, const int64_t *neighbors, int n,
                     int64_t n_entries, double cut2, int upper_only, uint8_t *keep, double *d2, void *stream) {
    if (n_entries == 0) return 0;
    filter_table_kernel<<<kf_blocks(n_entries, 256), 256, 0, (cudaStream_t)stream>>>(
        pos, offsets, neighbors, n, n_entries, cut2, upper_only, keep, d2);
    KF_LAUNCH_CHECK("filter_table_kernel");
    return 0;
}

int kf_compact_pairs(const int64_t *offsets, const int64_t *neighbors, int n, int64_t n_entries,
                     const uint8_t *keep, const double *d2, int64_t *dest /* [n_entries+1] */,
                     int64_t *scratch /* [n_entries] + 1024 */, int64_t *oi, int64_t *oj, double *od,
                     void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (kf_u8_to_i64_launch(keep, n_entries, scratch, s)) return 1;
    if (kf_scan_i64(scratch, n_entries, dest, scratch + n_entries, s)) return 1;
    if (n_entries == 0) return 0;
    compact_pairs_kernel<<<kf_blocks(n_entries, 256), 256, 0, s>>>(offsets, neighbors, n, n_entries, keep, dest,
                                                                   d2, oi, oj, od);
    KF_LAUNCH_CHECK("compact_pairs_kernel");
    return 0;
}

int kf_classify_pairs(const kf_field_t *f, const int64_t *i, const int64_t *j, int64_t n, int64_t *cls,
                      void *stream) {
    if (n == 0) return 0;
    classify_kernel<<<kf_blocks(n, 256), 256, 0, (cudaStream_t)stream>>>(*f, i, j, n, cls);
    KF_LAUNCH_CHECK("classify_kernel");
    return 0;
}

int kf_pair_terms(const kf_field_t *f, const double *pos, int n, const int64_t *i, const int64_t *j,
                  const double *d, const double *w, int64_t n_pairs, int kind, double *e_pair, double *mag,
                  double *forces, void *stream) {
    if (n_pairs == 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    double *fvec = nullptr;
    if (forces) KF_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&fvec), sizeof(double) * 3 * n_pairs, s), "fvec");
    pair_terms_kernel<<<kf_blocks(n_pairs, 256), 256, 0, s>>>(*f, pos, i, j, d, w, n_pairs, kind, e_pair, mag, fvec);
    KF_LAUNCH_CHECK("pair_terms_kernel");
    if (!forces) return 0;
    const int rc = scatter_bincount(n, i, j, n_pairs, fvec, forces, s);
    KF_CUDA(cudaFreeAsync(fvec, s), "fvec free");
    return rc;
}

int kf_scatter_pair_forces(const double *pos, int n, const int64_t *i, const int64_t *j, const double *d,
                           const double *mag, int64_t m, double *forces, void *stream) {
    if (m == 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    double *fvec = nullptr;
    KF_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&fvec), sizeof(double) * 3 * m, s), "fvec");
    pair_fvec_kernel<<<kf_blocks(m, 256), 256, 0, s>>>(pos, i, j, d, mag, m, fvec);
    KF_LAUNCH_CHECK("pair_fvec_kernel");
    const int rc = scatter_bincount(n, i, j, m, fvec, forces, s);
    KF_CUDA(cudaFreeAsync(fvec, s), "fvec free");
    return rc;
}

int kf_grid_occupied(const int32_t *counts, const int64_t *starts, int64_t n_keys, int64_t *scratch,
                     int64_t *dest, int64_t *occupied, int64_t *occ_starts, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (n_keys > 0) {
        nonzero_flags_kernel<<<kf_blocks(n_keys, 256), 256, 0, s>>>(counts, n_keys, scratch);
        KF_LAUNCH_CHECK("nonzero_flags_kernel");
    }
    if (kf_scan_i64(scratch, n_keys, dest, scratch + n_keys, s)) return 1;
    if (n_keys > 0) {
        occupied_kernel<<<kf_blocks(n_keys, 256), 256, 0, s>>>(counts, starts, dest, n_keys, occupied, occ_starts);
        KF_LAUNCH_CHECK("occupied_kernel");
    }
    return 0;
}

int kf_row_kept_offsets(const int64_t *offsets, int n, const int64_t *dest, int64_t *out, void *stream) {
    row_kept_kernel<<<kf_blocks(n + 1, 256), 256, 0, (cudaStream_t)stream>>>(offsets, n, dest, out);
    KF_LAUNCH_CHECK("row_kept_kernel");
    return 0;
}

int kf_argmin_f64(const double *x, int64_t m, int64_t *out, void *stream) {
    argmin_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(x, m, out);
    KF_LAUNCH_CHECK("argmin_kernel");
    return 0;
}

int kf_sum_f64(const double *x, int64_t n, double *partials, double *out, void *stream) {
    return kf_sum_f64_launch(x, n, partials, out, (cudaStream_t)stream);
}

int kf_scan_exclusive_i64(const int64_t *in, int64_t n, int64_t *out, int64_t *scratch, void *stream) {
    return kf_scan_i64(in, n, out, scratch, (cudaStream_t)stream);
}

}  // extern "C"
