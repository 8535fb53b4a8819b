// Spatial binning (K1) for the hot path.
//
// Reference: spatial.build_grid (/root/reference/pkg/src/kinefold/spatial.py:
// 83-114) sizes cells from the bounding box (~alpha*n cells) and the pair sets
// are filtered exactly afterwards (spatial.py:233-241), so any superset grid
// gives bit-identical pairs.  The hot path therefore bins on
// a fixed cell edge >= the largest interaction reach (9 A: a 27-cell stencil)
// into a per-trajectory open-addressing table with ONE slot per occupied cell:
// no bounding-box reduction, no host round trip, and a probe either finds the
// cell or proves it empty, so stencil walks never see foreign atoms.
//
//   insert   per atom: cell key -> CAS into the table (linear probing), the
//            first inserter appends the slot to the trajectory's occupied list,
//            rank = warp-aggregated atomicAdd on the slot count
//   scan     per trajectory: starts of occupied cells (list order) and the
//            work-item prefix over trajectories
//   scatter  sorted_atom[start + rank] = atom
//   finalize per occupied cell: members sorted by atom index (deterministic
//            visit order) and the cell-ordered SoA the pair kernel stages:
//            fp32 offset from the cell centre, fp64 position, params, aux ints
#include <algorithm>

#include "kf_common.cuh"

namespace {

constexpr int CELL_LIM = (1 << 20) - 2;
constexpr unsigned long long EMPTY = ~0ull;

KF_DEV int cell_coord(double x, double inv_cell) {
    double c = floor(x * inv_cell);
    c = fmin(fmax(c, (double)-CELL_LIM), (double)CELL_LIM);
    return (int)c;
}

__global__ void bin_insert_kernel(kf_field_t f, int B, int n, const double *__restrict__ pos,
                                  unsigned long long *__restrict__ keys, int32_t *__restrict__ cnt,
                                  int32_t *__restrict__ occ, int32_t *__restrict__ occ_count,
                                  int32_t *__restrict__ atom_slot, int32_t *__restrict__ atom_rank,
                                  kf_status_t *status) {
    kf_pdl_wait();      // after the predecessor (programmatic launch: single trajectories)
    kf_pdl_trigger();
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
    const unsigned long long key = (unsigned long long)pack_cell(cx, cy, cz);
    unsigned long long *tk = keys + (size_t)b * H;
    uint32_t slot = cell_hash(cx, cy, cz, H - 1);
    // warp leaders insert each distinct key once
    const unsigned active = __activemask();
    const unsigned same = __match_any_sync(active, key) & __match_any_sync(active, b);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(same) - 1;
    if (lane == leader) {
        for (;;) {
            const unsigned long long prev = atomicCAS(&tk[slot], EMPTY, key);
            if (prev == EMPTY) {
                occ[(size_t)b * H + atomicAdd(&occ_count[b], 1)] = (int32_t)slot;
                break;
            }
            if (prev == key) break;
            slot = (slot + 1) & (H - 1);
        }
    }
    slot = __shfl_sync(same, slot, leader);
    const int rank_in = __popc(same & ((1u << lane) - 1u));
    int base = 0;
    if (lane == leader) base = atomicAdd(&cnt[(size_t)b * H + slot], __popc(same));
    base = __shfl_sync(same, base, leader);
    atom_slot[gid] = (int32_t)slot;
    atom_rank[gid] = base + rank_in;
}

// Block-wide exclusive scan of one int per thread (blockDim a multiple of 32).
__device__ __forceinline__ int block_excl_scan(int v, int *wsum) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    __syncthreads();
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int t = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += u;
        }
        wsum[lane] = t;
    }
    __syncthreads();
    return incl - v + (wid > 0 ? wsum[wid - 1] : 0);
}

// Per trajectory: exclusive scans, in occupied-list order, of the cells' atom
// counts (-> cell_start, by slot) and of their 32-atom i-chunks (-> chunk_pre,
// by list position; the pair kernel's work items are (cell, i-chunk)).
__global__ void __launch_bounds__(1024)
cell_scan_kernel(int H, int chunk, const int32_t *__restrict__ occ, const int32_t *__restrict__ occ_count,
                 const int32_t *__restrict__ cnt, int32_t *__restrict__ start, int32_t *__restrict__ chunk_pre,
                 int32_t *__restrict__ item_cell, int32_t *__restrict__ chunk_count, const kf_status_t *status,
                 int32_t *__restrict__ occ_offset, int32_t *__restrict__ chunk_offset) {
    kf_pdl_wait();      // after the predecessor (programmatic launch: single trajectories)
    kf_pdl_trigger();
    // occ_offset / chunk_offset non-null (one trajectory): the work prefixes are
    // written here and occ_prefix_kernel is skipped
    const int b = blockIdx.x;
    if (status[b].done) {
        if (occ_offset && threadIdx.x == 0) { occ_offset[0] = occ_offset[1] = 0; chunk_offset[0] = chunk_offset[1] = 0; }
        return;
    }
    const int m = occ_count[b];
    const int32_t *ob = occ + (size_t)b * H;
    const int32_t *cb = cnt + (size_t)b * H;
    int32_t *sb = start + (size_t)b * H;
    int32_t *pb = chunk_pre + (size_t)b * H;
    const int per = (m + blockDim.x - 1) / blockDim.x;
    const int lo = min(m, (int)threadIdx.x * per), hi = min(m, lo + per);
    int local = 0, lchunk = 0;
    for (int k = lo; k < hi; ++k) {
        const int c = cb[ob[k]];
        local += c;
        lchunk += (c + chunk - 1) / chunk;
    }
    __shared__ int wsum[32];
    int run = block_excl_scan(local, wsum);
    int crun = block_excl_scan(lchunk, wsum);
    int32_t *ib = item_cell + (size_t)b * H;
    for (int k = lo; k < hi; ++k) {
        const int c = cb[ob[k]], nc = (c + chunk - 1) / chunk;
        sb[ob[k]] = run; run += c;
        pb[k] = crun;
        for (int q = 0; q < nc; ++q) ib[crun + q] = k;
        crun += nc;
    }
    if (threadIdx.x == blockDim.x - 1) {
        chunk_count[b] = crun;
        if (occ_offset) { occ_offset[0] = 0; occ_offset[1] = m; chunk_offset[0] = 0; chunk_offset[1] = crun; }
    }
}

// The per-launch hash-table reset (keys empty, counts and occupied counts zero):
// one kernel node instead of three memsets.
__global__ void bin_clear_kernel(long long n_tab, int B, unsigned long long *__restrict__ keys,
                                 int32_t *__restrict__ cnt, int32_t *__restrict__ occ_count) {
    kf_pdl_wait();      // after the predecessor (programmatic launch: single trajectories)
    kf_pdl_trigger();
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n_tab;
         q += (long long)gridDim.x * blockDim.x) {
        keys[q] = EMPTY;
        cnt[q] = 0;
        if (q < B) occ_count[q] = 0;
    }
}

// Work-item prefixes over trajectories: occupied cells (bin_finalize) and
// i-chunks (pair kernel).
__global__ void __launch_bounds__(1024)
occ_prefix_kernel(int B, const int32_t *__restrict__ occ_count, int32_t *__restrict__ occ_offset,
                  const int32_t *__restrict__ chunk_count, int32_t *__restrict__ chunk_offset,
                  const kf_status_t *status) {
    __shared__ int carry[2];
    __shared__ int ws[32];
    if (threadIdx.x == 0) carry[0] = carry[1] = 0;
    __syncthreads();
    for (int base = 0; base < B; base += blockDim.x) {
        const int b = base + threadIdx.x;
        const bool live = b < B && !status[b].done;
        const int v = live ? occ_count[b] : 0, u = live ? chunk_count[b] : 0;
        const int ev = carry[0] + block_excl_scan(v, ws);
        const int eu = carry[1] + block_excl_scan(u, ws);
        if (b < B) { occ_offset[b] = ev; chunk_offset[b] = eu; }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) { carry[0] = ev + v; carry[1] = eu + u; }
        __syncthreads();
    }
    if (threadIdx.x == 0) { occ_offset[B] = carry[0]; chunk_offset[B] = carry[1]; }
}

__global__ void bin_scatter_kernel(kf_field_t f, int B, int n, const int32_t *__restrict__ atom_slot,
                                   const int32_t *__restrict__ atom_rank, const int32_t *__restrict__ start,
                                   int32_t *__restrict__ sorted_atom, const kf_status_t *status) {
    kf_pdl_wait();      // after the predecessor (programmatic launch: single trajectories)
    kf_pdl_trigger();
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (long long)B * n) return;
    const int b = (int)(gid / n), a = (int)(gid % n);
    if (status[b].done) return;
    const size_t H = (size_t)1 << f.hash_bits;
    sorted_atom[(size_t)b * n + start[b * H + atom_slot[gid]] + atom_rank[gid]] = a;
}

// One warp per occupied cell: members ranked by atom index in parallel
// (deterministic visit order), then the cell-ordered SoA gathered one atom per
// lane: fp32 hi/lo offsets from the cell centre, fp64 position, params, aux,
// the static class window, and the members' bounding box.
constexpr int FIN_WARPS = 4;
constexpr int FIN_CAP = 1024;

// One occupied cell, one warp: rank sort of its members by atom index, then the
// cell-ordered SoA and the members' bounding box.  buf: FIN_CAP ints of this warp.
KF_DEV void finalize_cell(const kf_field_t &f, int b, int n, size_t H, int slot, int lane, int *buf, int cap,
                          const double *__restrict__ pos, const unsigned long long *__restrict__ keys,
                          const int32_t *__restrict__ cnt, const int32_t *__restrict__ start,
                          int32_t *__restrict__ sorted_atom, float4 *__restrict__ s_hi, float4 *__restrict__ s_lo,
                          double4 *__restrict__ s_pos, float4 *__restrict__ s_par, int4 *__restrict__ s_aux,
                          int4 *__restrict__ s_tree, float4 *__restrict__ cell_box) {
    const int s0 = start[b * H + slot], c = cnt[b * H + slot];
    int32_t *ids = sorted_atom + (size_t)b * n + s0;
    if (c <= cap) {
        for (int k = lane; k < c; k += 32) buf[k] = ids[k];
        __syncwarp();
        for (int k = lane; k < c; k += 32) {
            const int v = buf[k];
            int rank = 0;
            for (int m = 0; m < c; ++m) rank += buf[m] < v;
            ids[rank] = v;
        }
    } else if (lane == 0) {   // pathological cell: serial insertion sort
        for (int k = 1; k < c; ++k) {
            const int v = ids[k];
            int m = k - 1;
            while (m >= 0 && ids[m] > v) { ids[m + 1] = ids[m]; --m; }
            ids[m + 1] = v;
        }
    }
    __syncwarp();
    int cx, cy, cz;
    unpack_cell((long long)keys[b * H + slot], cx, cy, cz);
    const double ctr[3] = {((double)cx + 0.5) * f.cell, ((double)cy + 0.5) * f.cell, ((double)cz + 0.5) * f.cell};
    const bool tree = !f.uniform_weights;
    float bl[3] = {INFINITY, INFINITY, INFINITY}, bh[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int k = lane; k < c; k += 32) {
        const int a = ids[k];
        const size_t ga = (size_t)b * n + a, gs = (size_t)b * n + s0 + k;
        const double x = pos[3 * ga], y = pos[3 * ga + 1], z = pos[3 * ga + 2];
        s_pos[gs] = make_double4(x, y, z, f.solvation ? f.r_off[a] : 0.0);   // w: R_off (solvation gather)
        // offset from the cell centre as an fp32 pair: hi + lo == the fp64 offset
        // to ~1e-14 A, so fp32 arithmetic on them recovers fp64-accurate
        // difference vectors without absolute coordinates
        const double r[3] = {x - ctr[0], y - ctr[1], z - ctr[2]};
        float h[3], l[3];
        for (int q = 0; q < 3; ++q) {
            h[q] = (float)r[q];
            l[q] = (float)(r[q] - (double)h[q]);
            bl[q] = fminf(bl[q], h[q]);
            bh[q] = fmaxf(bh[q], h[q]);
        }
        s_hi[gs] = make_float4(h[0], h[1], h[2], 0.f);
        s_lo[gs] = make_float4(l[0], l[1], l[2], 0.f);
        s_par[gs] = reinterpret_cast<const float4 *>(f.atom_par)[a];
        s_aux[gs] = reinterpret_cast<const int4 *>(f.atom_aux)[a];
        s_tree[gs] = tree ? reinterpret_cast<const int4 *>(f.class_map)[a] : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1)
        for (int q = 0; q < 3; ++q) {
            bl[q] = fminf(bl[q], __shfl_xor_sync(0xffffffffu, bl[q], d));
            bh[q] = fmaxf(bh[q], __shfl_xor_sync(0xffffffffu, bh[q], d));
        }
    if (lane == 0) {
        cell_box[2 * (b * H + slot)] = make_float4(bl[0], bl[1], bl[2], 0.f);
        cell_box[2 * (b * H + slot) + 1] = make_float4(bh[0], bh[1], bh[2], 0.f);
    }
}

__global__ void __launch_bounds__(FIN_WARPS * 32)
bin_finalize_kernel(const __grid_constant__ kf_field_t f, int B, int n, const double *__restrict__ pos,
                    const unsigned long long *__restrict__ keys, const int32_t *__restrict__ occ,
                    const int32_t *__restrict__ occ_offset, const int32_t *__restrict__ cnt,
                    const int32_t *__restrict__ start, int32_t *__restrict__ sorted_atom,
                    float4 *__restrict__ s_hi, float4 *__restrict__ s_lo,
                    double4 *__restrict__ s_pos, float4 *__restrict__ s_par,
                    int4 *__restrict__ s_aux, int4 *__restrict__ s_tree,
                    float4 *__restrict__ cell_box, const kf_status_t *status) {
    kf_pdl_wait();      // after the predecessor (programmatic launch: single trajectories)
    kf_pdl_trigger();
    __shared__ int buf[FIN_WARPS][FIN_CAP];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int total = occ_offset[B];
    const size_t H = (size_t)1 << f.hash_bits;
    // persistent: warps stride over the occupied cells of all trajectories
    for (int item = blockIdx.x * FIN_WARPS + warp; item < total; item += gridDim.x * FIN_WARPS) {
        const int b = item_owner(occ_offset, B, item);
        const int slot = occ[b * H + (item - occ_offset[b])];
        finalize_cell(f, b, n, H, slot, lane, buf[warp], FIN_CAP, pos, keys, cnt, start, sorted_atom, s_hi, s_lo, s_pos,
                      s_par, s_aux, s_tree, cell_box);
        __syncwarp();
    }
}

// The last CTA of a per-trajectory binning kernel (ticket in work[2]) builds the
// work-item prefixes over trajectories (live ones only) from the published counts.
KF_DEV void publish_prefixes(int B, const int32_t *occ_count, const int32_t *chunk_count, int32_t *occ_offset,
                             int32_t *chunk_offset, int32_t *ticket, const kf_status_t *status, int *wsum) {
    __shared__ int last_s, carry_s[2];
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last_s = atomicAdd(ticket, 1) == B - 1;
    }
    __syncthreads();
    if (!last_s) return;
    __threadfence();
    if (threadIdx.x == 0) carry_s[0] = carry_s[1] = 0;
    __syncthreads();
    for (int base = 0; base < B; base += blockDim.x) {
        const int bb = base + threadIdx.x;
        const bool live = bb < B && !status[bb].done;
        const int v = live ? __ldcg(&occ_count[bb]) : 0, u = live ? __ldcg(&chunk_count[bb]) : 0;
        const int ev = carry_s[0] + block_excl_scan(v, wsum);
        const int eu = carry_s[1] + block_excl_scan(u, wsum);
        if (bb < B) { occ_offset[bb] = ev; chunk_offset[bb] = eu; }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) { carry_s[0] = ev + v; carry_s[1] = eu + u; }
        __syncthreads();
    }
    if (threadIdx.x == 0) { occ_offset[B] = carry_s[0]; chunk_offset[B] = carry_s[1]; *ticket = 0; }
}

// ---- small trajectories: the whole binning of one trajectory in one CTA -------
// Same table, scans, scatter and finalize as the kernel pipeline above, with
// block barriers in place of kernel boundaries and the table cleared by its own
// CTA (no memsets).  The last CTA to finish (ticket in work[2]) builds the
// work-item prefixes over trajectories from the published counts.
constexpr int BF_THREADS = 512;    // many trajectories: 4 CTAs per SM
constexpr int BF_THREADS_FEW = 1024;   // < 256 trajectories (about one CTA per SM): wider CTAs
constexpr int BF_FEW_B = 256;
#ifndef BF_MIN_B
#define BF_MIN_B 32   // trajectories from which binning runs fused (one CTA each)
#endif
#ifndef BF_MAX_ATOMS
#define BF_MAX_ATOMS 8192   // per-trajectory atoms below which binning runs fused
#endif
// per-warp rank-sort buffer (larger cells: serial insertion sort): 32 KB per CTA either way
template <int NT> constexpr int bf_cap() { return NT >= 1024 ? 256 : 512; }

template <int NT>
__global__ void __launch_bounds__(NT)
bin_fused_kernel(const __grid_constant__ kf_field_t f, int B, int n, int chunk, const double *__restrict__ pos,
                 unsigned long long *__restrict__ keys, int32_t *__restrict__ cnt, int32_t *__restrict__ start,
                 int32_t *__restrict__ occ, int32_t *__restrict__ occ_count, int32_t *__restrict__ chunk_pre,
                 int32_t *__restrict__ item_cell, int32_t *__restrict__ chunk_count, int32_t *__restrict__ occ_offset,
                 int32_t *__restrict__ chunk_offset, int32_t *__restrict__ atom_slot,
                 int32_t *__restrict__ atom_rank, int32_t *__restrict__ sorted_atom, float4 *__restrict__ s_hi,
                 float4 *__restrict__ s_lo, double4 *__restrict__ s_pos, float4 *__restrict__ s_par,
                 int4 *__restrict__ s_aux, int4 *__restrict__ s_tree, float4 *__restrict__ cell_box,
                 int32_t *__restrict__ ticket, kf_status_t *status) {
    __shared__ int m_s;
    __shared__ int wsum[32];
    constexpr int NWB = NT / 32, CAP = bf_cap<NT>();
    __shared__ int buf[NWB][CAP];
    // the trajectory's hash table (keys, then counts) in shared memory: the CAS
    // inserts and the warp-aggregated counts are shared-memory atomics; the table is
    // written out once, coalesced, for the later kernels (solvation, pairs)
    extern __shared__ __align__(16) unsigned char bf_dyn[];
    const int b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t H = (size_t)1 << f.hash_bits;
    unsigned long long *sk = reinterpret_cast<unsigned long long *>(bf_dyn);
    int32_t *sc = reinterpret_cast<int32_t *>(sk + H);
    if (!status[b].done) {
        unsigned long long *tk = keys + b * H;
        int32_t *tc = cnt + b * H, *ts = start + b * H, *to = occ + b * H, *tp = chunk_pre + b * H;
        for (size_t q = threadIdx.x; q < H; q += blockDim.x) { sk[q] = EMPTY; sc[q] = 0; }
        if (threadIdx.x == 0) m_s = 0;
        __syncthreads();
        // insert: cell key per atom, CAS into the table, warp-aggregated counts
        const double inv = 1.0 / f.cell;
        for (int a0 = 0; a0 < n; a0 += blockDim.x) {
            const int a = a0 + threadIdx.x;
            if (a < n) {
                const size_t ga = (size_t)b * n + a;
                const double x = pos[3 * ga], y = pos[3 * ga + 1], z = pos[3 * ga + 2];
                int cx = 0, cy = 0, cz = 0;
                if (!(isfinite(x) && isfinite(y) && isfinite(z))) {
                    if (atomicCAS(&status[b].error, KF_ERR_NONE, KF_ERR_NONFINITE) == KF_ERR_NONE)
                        status[b].err_iter = status[b].iter;
                } else {
                    cx = cell_coord(x, inv); cy = cell_coord(y, inv); cz = cell_coord(z, inv);
                }
                const unsigned long long key = (unsigned long long)pack_cell(cx, cy, cz);
                uint32_t slot = cell_hash(cx, cy, cz, (uint32_t)H - 1);
                const unsigned active = __activemask();
                const unsigned same = __match_any_sync(active, key);
                const int leader = __ffs(same) - 1;
                if (lane == leader) {
                    for (;;) {
                        const unsigned long long prev = atomicCAS(&sk[slot], EMPTY, key);
                        if (prev == EMPTY) { to[atomicAdd(&m_s, 1)] = (int32_t)slot; break; }
                        if (prev == key) break;
                        slot = (slot + 1) & ((uint32_t)H - 1);
                    }
                }
                slot = __shfl_sync(same, slot, leader);
                const int rank_in = __popc(same & ((1u << lane) - 1u));
                int base = 0;
                if (lane == leader) base = atomicAdd(&sc[slot], __popc(same));
                base = __shfl_sync(same, base, leader);
                atom_slot[ga] = (int32_t)slot;
                atom_rank[ga] = base + rank_in;
            }
        }
        __syncthreads();
        for (size_t q = threadIdx.x; q < H; q += blockDim.x) { tk[q] = sk[q]; tc[q] = sc[q]; }
        // exclusive scans of atom counts and i-chunks over the occupied list
        const int m = m_s;
        const int per = (m + blockDim.x - 1) / blockDim.x;
        const int lo = min(m, (int)threadIdx.x * per), hi = min(m, lo + per);
        int local = 0, lchunk = 0;
        for (int k = lo; k < hi; ++k) {
            const int c = sc[to[k]];
            local += c;
            lchunk += (c + chunk - 1) / chunk;
        }
        int run = block_excl_scan(local, wsum);
        int crun = block_excl_scan(lchunk, wsum);
        int32_t *ti = item_cell + b * H;
        for (int k = lo; k < hi; ++k) {
            const int c = sc[to[k]], nc = (c + chunk - 1) / chunk;
            ts[to[k]] = run; run += c;
            tp[k] = crun;
            for (int q = 0; q < nc; ++q) ti[crun + q] = k;
            crun += nc;
        }
        if (threadIdx.x == blockDim.x - 1) { occ_count[b] = m; chunk_count[b] = crun; }
        __syncthreads();
        // scatter, then one warp per cell
        for (int a = threadIdx.x; a < n; a += blockDim.x) {
            const size_t ga = (size_t)b * n + a;
            sorted_atom[(size_t)b * n + ts[atom_slot[ga]] + atom_rank[ga]] = a;
        }
        __syncthreads();
        for (int k = warp; k < m; k += NWB) {
            finalize_cell(f, b, n, H, to[k], lane, buf[warp], CAP, pos, keys, cnt, start, sorted_atom, s_hi, s_lo, s_pos,
                          s_par, s_aux, s_tree, cell_box);
            __syncwarp();
        }
    }
    publish_prefixes(B, occ_count, chunk_count, occ_offset, chunk_offset, ticket, status, wsum);
}


// ---- FieldConfig(use_hash=False): the quadratic all-pairs layout ---------------
// Reference: Field._neighbor_table -> _brute_table (kcm.py:94-102, :153-162):
// every pair is a candidate, no hashing.  Here: ONE cell holding every atom in
// index order (identity permutation, no sort), centred on the trajectory's
// centroid, with the one-cell stencil {0,0,0} (host side), so the same pair and
// solvation kernels sweep all n^2 / 2 candidates.  The fp32 hi offsets must stay
// within FLAT_MAX_OFFSET of the centre for the 1e-2 A^2 prefilter margin
// (ulp(2048) = 1.2e-4 A -> |d(d^2)| < 8e-3 A^2 at the 9 A cut-off); beyond it the
// trajectory stops with KF_ERR_EXTENT.  One CTA per trajectory.
constexpr int FL_THREADS = 512;
constexpr double FLAT_MAX_OFFSET = 2048.0;

__global__ void __launch_bounds__(FL_THREADS)
bin_flat_kernel(const __grid_constant__ kf_field_t f, int B, int n, int chunk, const double *__restrict__ pos,
                unsigned long long *__restrict__ keys, int32_t *__restrict__ cnt, int32_t *__restrict__ start,
                int32_t *__restrict__ occ, int32_t *__restrict__ occ_count, int32_t *__restrict__ chunk_pre,
                int32_t *__restrict__ item_cell, int32_t *__restrict__ chunk_count, int32_t *__restrict__ occ_offset,
                int32_t *__restrict__ chunk_offset, int32_t *__restrict__ atom_slot,
                int32_t *__restrict__ atom_rank, int32_t *__restrict__ sorted_atom, float4 *__restrict__ s_hi,
                float4 *__restrict__ s_lo, double4 *__restrict__ s_pos, float4 *__restrict__ s_par,
                int4 *__restrict__ s_aux, int4 *__restrict__ s_tree, float4 *__restrict__ cell_box,
                int32_t *__restrict__ ticket, kf_status_t *status) {
    constexpr int NWF = FL_THREADS / 32;
    __shared__ double red_s[NWF][3];
    __shared__ float box_s[NWF][6];
    __shared__ int slot_s, cell_s[3];
    __shared__ int wsum[32];
    const int b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t H = (size_t)1 << f.hash_bits;
    if (!status[b].done) {
        const double *pb = pos + (size_t)b * n * 3;
        // centroid of the finite coordinates (fixed reduction order)
        double sx = 0.0, sy = 0.0, sz = 0.0;
        int bad = 0;
        for (int a = threadIdx.x; a < n; a += blockDim.x) {
            const double x = pb[3 * a], y = pb[3 * a + 1], z = pb[3 * a + 2];
            if (isfinite(x) && isfinite(y) && isfinite(z)) { sx += x; sy += y; sz += z; } else bad = 1;
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            sx += __shfl_xor_sync(0xffffffffu, sx, d);
            sy += __shfl_xor_sync(0xffffffffu, sy, d);
            sz += __shfl_xor_sync(0xffffffffu, sz, d);
        }
        if (lane == 0) { red_s[warp][0] = sx; red_s[warp][1] = sy; red_s[warp][2] = sz; }
        bad = __syncthreads_or(bad);
        if (bad && threadIdx.x == 0 && atomicCAS(&status[b].error, KF_ERR_NONE, KF_ERR_NONFINITE) == KF_ERR_NONE)
            status[b].err_iter = status[b].iter;
        unsigned long long *tk = keys + b * H;
        int32_t *tc = cnt + b * H;
        for (size_t q = threadIdx.x; q < H; q += blockDim.x) { tk[q] = EMPTY; tc[q] = 0; }
        __syncthreads();
        if (threadIdx.x == 0) {
            double c[3] = {0.0, 0.0, 0.0};
            for (int w = 0; w < NWF; ++w)
                for (int q = 0; q < 3; ++q) c[q] += red_s[w][q];
            const double inv = 1.0 / f.cell;
            const int cx = cell_coord(c[0] / n, inv), cy = cell_coord(c[1] / n, inv), cz = cell_coord(c[2] / n, inv);
            const uint32_t slot = cell_hash(cx, cy, cz, (uint32_t)H - 1);
            tk[slot] = (unsigned long long)pack_cell(cx, cy, cz);
            tc[slot] = n;
            start[b * H + slot] = 0;
            occ[b * H] = (int32_t)slot;
            chunk_pre[b * H] = 0;
            occ_count[b] = 1;
            chunk_count[b] = (n + chunk - 1) / chunk;
            slot_s = (int)slot; cell_s[0] = cx; cell_s[1] = cy; cell_s[2] = cz;
        }
        __syncthreads();
        const int slot = slot_s;
        const double ctr[3] = {((double)cell_s[0] + 0.5) * f.cell, ((double)cell_s[1] + 0.5) * f.cell,
                               ((double)cell_s[2] + 0.5) * f.cell};
        for (int q = threadIdx.x; q < (n + chunk - 1) / chunk; q += blockDim.x) item_cell[b * H + q] = 0;
        const bool tree = !f.uniform_weights;
        float bl[3] = {INFINITY, INFINITY, INFINITY}, bh[3] = {-INFINITY, -INFINITY, -INFINITY};
        int far = 0;
        for (int a = threadIdx.x; a < n; a += blockDim.x) {
            const size_t g = (size_t)b * n + a;
            const double x = pb[3 * a], y = pb[3 * a + 1], z = pb[3 * a + 2];
            atom_slot[g] = slot; atom_rank[g] = a; sorted_atom[g] = a;
            s_pos[g] = make_double4(x, y, z, f.solvation ? f.r_off[a] : 0.0);
            const double r[3] = {x - ctr[0], y - ctr[1], z - ctr[2]};
            float h[3], l[3];
            for (int q = 0; q < 3; ++q) {
                h[q] = (float)r[q];
                l[q] = (float)(r[q] - (double)h[q]);
                bl[q] = fminf(bl[q], h[q]);
                bh[q] = fmaxf(bh[q], h[q]);
                far |= !(fabs(r[q]) <= FLAT_MAX_OFFSET);
            }
            s_hi[g] = make_float4(h[0], h[1], h[2], 0.f);
            s_lo[g] = make_float4(l[0], l[1], l[2], 0.f);
            s_par[g] = reinterpret_cast<const float4 *>(f.atom_par)[a];
            s_aux[g] = reinterpret_cast<const int4 *>(f.atom_aux)[a];
            s_tree[g] = tree ? reinterpret_cast<const int4 *>(f.class_map)[a] : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1)
            for (int q = 0; q < 3; ++q) {
                bl[q] = fminf(bl[q], __shfl_xor_sync(0xffffffffu, bl[q], d));
                bh[q] = fmaxf(bh[q], __shfl_xor_sync(0xffffffffu, bh[q], d));
            }
        if (lane == 0)
            for (int q = 0; q < 3; ++q) { box_s[warp][q] = bl[q]; box_s[warp][3 + q] = bh[q]; }
        far = __syncthreads_or(far);
        if (threadIdx.x == 0) {
            for (int w = 1; w < NWF; ++w)
                for (int q = 0; q < 3; ++q) {
                    box_s[0][q] = fminf(box_s[0][q], box_s[w][q]);
                    box_s[0][3 + q] = fmaxf(box_s[0][3 + q], box_s[w][3 + q]);
                }
            cell_box[2 * (b * H + slot)] = make_float4(box_s[0][0], box_s[0][1], box_s[0][2], 0.f);
            cell_box[2 * (b * H + slot) + 1] = make_float4(box_s[0][3], box_s[0][4], box_s[0][5], 0.f);
            if (far && !bad && atomicCAS(&status[b].error, KF_ERR_NONE, KF_ERR_EXTENT) == KF_ERR_NONE)
                status[b].err_iter = status[b].iter;
        }
    }
    publish_prefixes(B, occ_count, chunk_count, occ_offset, chunk_offset, ticket, status, wsum);
}

}  // namespace

int kf_cluster_path(const kf_field_t *f, const kf_batch_t *w, int n);

int kf_bin_launch(const kf_field_t *f, kf_batch_t *w, int n, cudaStream_t s) {
    // the cluster-pair kernel needs no cell table; only the solvation pass does
    if (!f->solvation && kf_cluster_path(f, w, n)) return 0;
    const int B = w->B, H = 1 << f->hash_bits;
    if (f->flat) {   // FieldConfig(use_hash=False)
        bin_flat_kernel<<<B, FL_THREADS, 0, s>>>(
            *f, B, n, kf_pair_chunk(B, n, w->pair_chunk, f->precision), w->pos, w->cell_key, w->cell_cnt,
            w->cell_start, w->occ, w->occ_count, w->chunk_pre, w->item_cell, w->chunk_count, w->occ_offset, w->chunk_offset,
            w->atom_slot, w->atom_rank, w->sorted_atom, reinterpret_cast<float4 *>(w->s_hi),
            reinterpret_cast<float4 *>(w->s_lo), reinterpret_cast<double4 *>(w->s_pos),
            reinterpret_cast<float4 *>(w->s_par), reinterpret_cast<int4 *>(w->s_aux),
            reinterpret_cast<int4 *>(w->s_tree), reinterpret_cast<float4 *>(w->cell_box), w->work + 2, w->status);
        KF_LAUNCH_CHECK("bin_flat_kernel");
        return 0;
    }
    if (n <= BF_MAX_ATOMS && B >= BF_MIN_B) {   // ensembles: one CTA per trajectory does the whole binning
        auto kern = B < BF_FEW_B ? bin_fused_kernel<BF_THREADS_FEW> : bin_fused_kernel<BF_THREADS>;
        const size_t dyn = (size_t)H * (sizeof(unsigned long long) + sizeof(int32_t));   // the shared hash table
        static size_t opted[2] = {0, 0};
        const int few = B < BF_FEW_B;
        if (dyn > opted[few]) {
            KF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn), "bin smem");
            opted[few] = dyn;
        }
        kern<<<B, B < BF_FEW_B ? BF_THREADS_FEW : BF_THREADS, dyn, s>>>(
            *f, B, n, kf_pair_chunk(B, n, w->pair_chunk, f->precision), w->pos, w->cell_key, w->cell_cnt,
            w->cell_start, w->occ, w->occ_count, w->chunk_pre, w->item_cell, w->chunk_count, w->occ_offset, w->chunk_offset,
            w->atom_slot, w->atom_rank, w->sorted_atom, reinterpret_cast<float4 *>(w->s_hi),
            reinterpret_cast<float4 *>(w->s_lo), reinterpret_cast<double4 *>(w->s_pos),
            reinterpret_cast<float4 *>(w->s_par), reinterpret_cast<int4 *>(w->s_aux),
            reinterpret_cast<int4 *>(w->s_tree), reinterpret_cast<float4 *>(w->cell_box), w->work + 2, w->status);
        KF_LAUNCH_CHECK("bin_fused_kernel");
        return 0;
    }
    const long long n_tab = (long long)B * H;
    const bool pdl = B < KF_PDL_B;
    (void)kf_launch(pdl, bin_clear_kernel, dim3((unsigned)std::min<long long>(kf_blocks(n_tab, 256), 4 * 148)),
                    dim3(256), 0, s, n_tab, B, w->cell_key, w->cell_cnt, w->occ_count);
    KF_LAUNCH_CHECK("bin_clear_kernel");
    const long long total = (long long)B * n;
    (void)kf_launch(pdl, bin_insert_kernel, dim3(kf_blocks(total, 256)), dim3(256), 0, s, *f, B, n,
                    (const double *)w->pos, w->cell_key, w->cell_cnt, w->occ, w->occ_count, w->atom_slot,
                    w->atom_rank, w->status);
    KF_LAUNCH_CHECK("bin_insert_kernel");
    (void)kf_launch(pdl, cell_scan_kernel, dim3(B), dim3(1024), 0, s, H, kf_pair_chunk(B, n, w->pair_chunk, f->precision),
                    (const int32_t *)w->occ, (const int32_t *)w->occ_count, (const int32_t *)w->cell_cnt,
                    w->cell_start, w->chunk_pre, w->item_cell, w->chunk_count, (const kf_status_t *)w->status,
                    B == 1 ? w->occ_offset : (int32_t *)nullptr, B == 1 ? w->chunk_offset : (int32_t *)nullptr);
    KF_LAUNCH_CHECK("cell_scan_kernel");
    if (B > 1) {
        occ_prefix_kernel<<<1, 1024, 0, s>>>(B, w->occ_count, w->occ_offset, w->chunk_count, w->chunk_offset,
                                             w->status);
        KF_LAUNCH_CHECK("occ_prefix_kernel");
    }
    (void)kf_launch(pdl, bin_scatter_kernel, dim3(kf_blocks(total, 256)), dim3(256), 0, s, *f, B, n,
                    (const int32_t *)w->atom_slot, (const int32_t *)w->atom_rank, (const int32_t *)w->cell_start,
                    w->sorted_atom, (const kf_status_t *)w->status);
    KF_LAUNCH_CHECK("bin_scatter_kernel");
    static int fin_grid = 0;
    if (fin_grid == 0) {
        int dev = 0, sms = 148, per_sm = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bin_finalize_kernel, FIN_WARPS * 32, 0);
        fin_grid = sms * (per_sm > 0 ? per_sm : 1);
    }
    (void)kf_launch(pdl, bin_finalize_kernel, dim3((unsigned)std::min<long long>(fin_grid, kf_blocks(total, FIN_WARPS))),
        dim3(FIN_WARPS * 32), 0, s,
        *f, B, n, w->pos, w->cell_key, w->occ, w->occ_offset, w->cell_cnt, w->cell_start, w->sorted_atom,
        reinterpret_cast<float4 *>(w->s_hi), reinterpret_cast<float4 *>(w->s_lo),
        reinterpret_cast<double4 *>(w->s_pos), reinterpret_cast<float4 *>(w->s_par),
        reinterpret_cast<int4 *>(w->s_aux), reinterpret_cast<int4 *>(w->s_tree),
        reinterpret_cast<float4 *>(w->cell_box), w->status);
    KF_LAUNCH_CHECK("bin_finalize_kernel");
    return 0;
}
