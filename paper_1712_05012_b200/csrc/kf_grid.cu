// Spatial binning (K1) for the hot path: per-atom cell key, warp-aggregated
// bucket histogram, per-trajectory exclusive scan, scatter, and a
// deterministic in-bucket order (ascending atom index).
//
// Reference: spatial.build_grid (/root/reference/pkg/src/kinefold/spatial.py:
// 83-114).  The reference sizes cells from the bounding box (~alpha*n cells);
// its pair sets are filtered exactly afterwards (spatial.py:233-241), so any
// superset gives bit-identical pairs.  The hot path therefore
// bins on a fixed cell edge into a power-of-two hash table per trajectory —
// no bounding-box reduction and no host round trip inside the loop.  The
// reference grid itself (bit-exact cell_index / occupied / starts / order) is
// produced by the API kernels in kf_refgrid.cu.
#include "kf_common.cuh"

namespace {

constexpr int CELL_LIM = (1 << 20) - 1;

KF_DEV int cell_coord(double x, double inv_cell) {
    double c = floor(x * inv_cell);
    c = fmin(fmax(c, (double)-CELL_LIM), (double)CELL_LIM);
    return (int)c;
}

__global__ void bin_count_kernel(kf_field_t f, int B, int n, const double *__restrict__ pos,
                                 int32_t *__restrict__ atom_cell, int32_t *__restrict__ atom_slot,
                                 int32_t *__restrict__ bucket_count, kf_status_t *status) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (long long)B * n) return;
    const int b = (int)(gid / n);
    if (status[b].done) return;
    const uint32_t H = 1u << f.hash_bits;
    const double x = pos[3 * gid], y = pos[3 * gid + 1], z = pos[3 * gid + 2];
    int cx = 0, cy = 0, cz = 0;
    if (!(isfinite(x) && isfinite(y) && isfinite(z))) {
        if (atomicCAS(&status[b].error, KF_ERR_NONE, KF_ERR_NONFINITE) == KF_ERR_NONE)
            status[b].err_iter = status[b].iter;
    } else {
        const double inv = 1.0 / f.cell;
        cx = cell_coord(x, inv); cy = cell_coord(y, inv); cz = cell_coord(z, inv);
    }
    atom_cell[3 * gid] = cx; atom_cell[3 * gid + 1] = cy; atom_cell[3 * gid + 2] = cz;
    const uint32_t key = (uint32_t)b * H + cell_hash(cx, cy, cz, H - 1);
    // warp-aggregated atomics: consecutive chain atoms usually share a cell
    const unsigned active = __activemask();
    const unsigned peers = __match_any_sync(active, key);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    const int rank = __popc(peers & ((1u << lane) - 1u));
    int base = 0;
    if (lane == leader) base = atomicAdd(&bucket_count[key], __popc(peers));
    base = __shfl_sync(peers, base, leader);
    atom_slot[gid] = base + rank;
}

// Exclusive scan of each trajectory's bucket counts (one CTA per trajectory).
__global__ void __launch_bounds__(1024)
bucket_scan_kernel(int H, const int32_t *__restrict__ count, int32_t *__restrict__ start,
                   const kf_status_t *status) {
    const int b = blockIdx.x;
    if (status[b].done) return;
    const int32_t *cnt = count + (size_t)b * H;
    int32_t *out = start + (size_t)b * (H + 1);
    const int per = (H + blockDim.x - 1) / blockDim.x;
    const int lo = min(H, (int)threadIdx.x * per), hi = min(H, lo + per);
    int local = 0;
    for (int k = lo; k < hi; ++k) local += cnt[k];
    __shared__ int wsum[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int v = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        wsum[lane] = v;
    }
    __syncthreads();
    int run = incl - local + (wid > 0 ? wsum[wid - 1] : 0);
    for (int k = lo; k < hi; ++k) { out[k] = run; run += cnt[k]; }
    if (threadIdx.x == blockDim.x - 1) out[H] = run;
}

__global__ void bucket_scatter_kernel(kf_field_t f, int B, int n, const int32_t *__restrict__ atom_cell,
                                      const int32_t *__restrict__ atom_slot,
                                      const int32_t *__restrict__ start, int32_t *__restrict__ sorted_atom,
                                      const kf_status_t *status) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (long long)B * n) return;
    const int b = (int)(gid / n), a = (int)(gid % n);
    if (status[b].done) return;
    const uint32_t H = 1u << f.hash_bits;
    const uint32_t h = cell_hash(atom_cell[3 * gid], atom_cell[3 * gid + 1], atom_cell[3 * gid + 2], H - 1);
    sorted_atom[(size_t)b * n + start[(size_t)b * (H + 1) + h] + atom_slot[gid]] = a;
}

// Sort each bucket by atom index (buckets hold a few atoms) and gather the
// bucket-ordered coordinates with the packed cell in the 4th lane.
__global__ void bucket_finalize_kernel(kf_field_t f, int B, int n, const double *__restrict__ pos,
                                       const int32_t *__restrict__ atom_cell,
                                       const int32_t *__restrict__ start, int32_t *__restrict__ sorted_atom,
                                       double *__restrict__ sorted_pos, const kf_status_t *status) {
    const int H = 1 << f.hash_bits;
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (long long)B * H) return;
    const int b = (int)(gid / H), h = (int)(gid % H);
    if (status[b].done) return;
    const int s0 = start[(size_t)b * (H + 1) + h], s1 = start[(size_t)b * (H + 1) + h + 1];
    int32_t *ids = sorted_atom + (size_t)b * n;
    for (int k = s0 + 1; k < s1; ++k) {
        const int v = ids[k];
        int m = k - 1;
        while (m >= s0 && ids[m] > v) { ids[m + 1] = ids[m]; --m; }
        ids[m + 1] = v;
    }
    for (int k = s0; k < s1; ++k) {
        const size_t a = (size_t)b * n + ids[k];
        double4 v;
        v.x = pos[3 * a]; v.y = pos[3 * a + 1]; v.z = pos[3 * a + 2];
        v.w = __longlong_as_double(pack_cell(atom_cell[3 * a], atom_cell[3 * a + 1], atom_cell[3 * a + 2]));
        reinterpret_cast<double4 *>(sorted_pos)[(size_t)b * n + k] = v;
    }
}

}  // namespace

int kf_bin_launch(const kf_field_t *f, kf_batch_t *w, int n, cudaStream_t s) {
    const int B = w->B, H = 1 << f->hash_bits;
    KF_CUDA(cudaMemsetAsync(w->bucket_count, 0, sizeof(int32_t) * (size_t)B * H, s), "memset buckets");
    const long long total = (long long)B * n;
    bin_count_kernel<<<kf_blocks(total, 256), 256, 0, s>>>(*f, B, n, w->pos, w->atom_cell, w->atom_slot,
                                                           w->bucket_count, w->status);
    KF_LAUNCH_CHECK("bin_count_kernel");
    bucket_scan_kernel<<<B, 1024, 0, s>>>(H, w->bucket_count, w->bucket_start, w->status);
    KF_LAUNCH_CHECK("bucket_scan_kernel");
    bucket_scatter_kernel<<<kf_blocks(total, 256), 256, 0, s>>>(*f, B, n, w->atom_cell, w->atom_slot,
                                                                w->bucket_start, w->sorted_atom, w->status);
    KF_LAUNCH_CHECK("bucket_scatter_kernel");
    bucket_finalize_kernel<<<kf_blocks((long long)B * H, 256), 256, 0, s>>>(
        *f, B, n, w->pos, w->atom_cell, w->bucket_start, w->sorted_atom, w->sorted_pos, w->status);
    KF_LAUNCH_CHECK("bucket_finalize_kernel");
    return 0;
}
