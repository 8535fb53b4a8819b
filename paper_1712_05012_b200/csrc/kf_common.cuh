// Shared device helpers for the kfb200 kernels (sm_100a).
#pragma once
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include "kfb200.h"

#define KF_DEV __device__ __forceinline__

// ---- exact IEEE fp64 primitives ------------------------------------------
// The reference's parity-critical arithmetic (cutoff tests, coverage tests,
// angle wrapping) is numpy elementwise fp64 with no FMA contraction; these
// intrinsics pin each operation to one correctly rounded op.
KF_DEV double xadd(double a, double b) { return __dadd_rn(a, b); }
KF_DEV double xsub(double a, double b) { return __dsub_rn(a, b); }
KF_DEV double xmul(double a, double b) { return __dmul_rn(a, b); }

// np.einsum('ij,ij->i', d, d) association on the reference host:
// (dx*dx + dz*dz) + dy*dy (SURVEY.md §0.4; spatial.py:239, :252).
KF_DEV double d2_einsum(double dx, double dy, double dz) {
    return xadd(xadd(xmul(dx, dx), xmul(dz, dz)), xmul(dy, dy));
}
// (diff * diff).sum(-1) association: (dx*dx + dy*dy) + dz*dz
// (solvation.py:159, :229, :241).
KF_DEV double d2_rowsum(double dx, double dy, double dz) {
    return xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz));
}

// numpy float remainder: fmod, then shift into the divisor's sign, zeros -> +0.0
// (geometry.py:44-46 -> npy_remainder).
KF_DEV double np_mod360(double a) {
    double r = fmod(a, 360.0);
    if (r != 0.0) {
        if (r < 0.0) r = xadd(r, 360.0);
    } else {
        r = 0.0;
    }
    return r;
}

// ---- rigid transforms: [M row-major 3x3 | p], x -> M x + p ----------------
// link_T rows are KF_XF_STRIDE doubles: M (9), joint point P (3), axis U (3), pad
#define KF_XF_STRIDE 16
// Pair-kernel work items: occupied cells cut into i-chunks of at most `chunk`
// atoms (a power of two <= 32).  Small chunks keep the dense kernel's lanes busy
// (a chunk of c atoms runs 32 / c j-phases); large ones amortise the per-item
// neighbour staging over more atoms.  Measured optimum on B200 (C2 chains):
// 4 below 4k atoms per launch, 8 below 1M, 16 above; the fp64 pair mode (the
// compacted kernel, lane = one of 32 owners) keeps 32.  kf_batch_t.pair_chunk
// overrides (0 = this rule).  Part of the work decomposition, so results are
// bitwise reproducible for a given (B, n) but not across chunk sizes.
inline int kf_pair_chunk(int B, int n, int requested, int precision) {
    static int env_chunk = -1;   // KFB200_PAIR_CHUNK: process-wide override (measurements)
    if (env_chunk < 0) {
        const char *e = getenv("KFB200_PAIR_CHUNK");
        env_chunk = e ? atoi(e) : 0;
    }
    if (!requested) requested = env_chunk;
    if (requested == 4 || requested == 8 || requested == 16 || requested == 32) return requested;
    if (precision) return 32;
    const long long atoms = (long long)B * n;
    // measured on B200 (C2 chains, graph-replayed): ensembles of 128+ trajectories
    // run fastest with 16-atom items (B=128: 396k vs 375k traj-it/s at 8), 64 with 8
    return atoms < 4000 ? 4 : atoms < 150000 ? 8 : 16;
}


// Programmatic dependent launch (single trajectories): a kernel launched with
// kf_launch(pdl = true, ...) may be scheduled while its predecessor runs; it
// waits here for the predecessor's completion (and memory) before touching
// anything.  Both are no-ops for kernels launched without the attribute.
KF_DEV void kf_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
KF_DEV void kf_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

#ifndef KF_PDL_B
#define KF_PDL_B 64   // batches below this launch the iteration chain with PDL
#endif
template <typename... KArgs, typename... Args>
inline cudaError_t kf_launch(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid; cfg.blockDim = block; cfg.dynamicSmemBytes = smem; cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

struct Xf { double m[9]; double p[3]; };

KF_DEV Xf xf_identity() {
    Xf t;
#pragma unroll
    for (int k = 0; k < 9; ++k) t.m[k] = (k % 4 == 0) ? 1.0 : 0.0;
    t.p[0] = t.p[1] = t.p[2] = 0.0;
    return t;
}
// (a o b)(x) = a(b(x)): M = Ma Mb, p = Ma pb + pa
KF_DEV Xf xf_compose(const Xf &a, const Xf &b) {
    Xf r;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
        for (int j = 0; j < 3; ++j)
            r.m[3 * i + j] = a.m[3 * i] * b.m[j] + a.m[3 * i + 1] * b.m[3 + j] + a.m[3 * i + 2] * b.m[6 + j];
        r.p[i] = a.m[3 * i] * b.p[0] + a.m[3 * i + 1] * b.p[1] + a.m[3 * i + 2] * b.p[2] + a.p[i];
    }
    return r;
}
KF_DEV Xf xf_load(const double *s) {
    Xf t;
#pragma unroll
    for (int k = 0; k < 9; ++k) t.m[k] = s[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) t.p[k] = s[9 + k];
    return t;
}
KF_DEV void xf_store(double *d, const Xf &t) {
#pragma unroll
    for (int k = 0; k < 9; ++k) d[k] = t.m[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) d[9 + k] = t.p[k];
}

// ---- spatial hash ----------------------------------------------------------
KF_DEV uint32_t cell_hash(int cx, int cy, int cz, uint32_t mask) {
    uint32_t h = (uint32_t)cx * 0x8da6b343u ^ (uint32_t)cy * 0xd8163841u ^ (uint32_t)cz * 0xcb1ab31fu;
    h ^= h >> 15;
    return h & mask;
}
// 3 x 21-bit signed cell coordinates packed in 63 bits (exact for |c| < 2^20)
KF_DEV long long pack_cell(int cx, int cy, int cz) {
    const long long m = (1LL << 21) - 1;
    return ((long long)(cx & m) << 42) | ((long long)(cy & m) << 21) | (long long)(cz & m);
}

KF_DEV void unpack_cell(long long p, int &cx, int &cy, int &cz) {
    const unsigned long long u = (unsigned long long)p;
    cx = (int)((long long)(u << 1) >> 43);
    cy = (int)((long long)(u << 22) >> 43);
    cz = (int)((long long)(u << 43) >> 43);
}
// Slot of cell (cx, cy, cz) in a trajectory's open-addressing table, or -1.
KF_DEV int cell_probe(const unsigned long long *tk, uint32_t H, int cx, int cy, int cz) {
    const unsigned long long key = (unsigned long long)pack_cell(cx, cy, cz);
    uint32_t slot = cell_hash(cx, cy, cz, H - 1);
    for (;;) {
        const unsigned long long k = tk[slot];
        if (k == key) return (int)slot;
        if (k == ~0ull) return -1;
        slot = (slot + 1) & (H - 1);
    }
}
// Trajectory owning work item `item` given the exclusive prefix off[0..B].
KF_DEV int item_owner(const int32_t *off, int B, int item) {
    int lo = 0, hi = B;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= item) lo = mid; else hi = mid;
    }
    return lo;
}

// Interaction class 1..4 (topology.py:153-178): tree neighbours only when both
// atoms are chain atoms within one residue of each other; 1-2 beats 1-3 beats 1-4.
KF_DEV int classify_pair(const kf_field_t &f, int i, int j, int pi, int gpi, int ggi, int ri, bool ci) {
    if (!ci || !f.tchain[j]) return 4;
    const int rj = f.tres[j];
    if (abs(ri - rj) > 1) return 4;
    const int pj = f.tparent[j], gpj = f.tgp[j], ggj = f.tggp[j];
    if (pi == j || pj == i) return 1;
    if (gpi == j || gpj == i || (pi >= 0 && pi == pj)) return 2;
    if (ggi == j || ggj == i || (gpi >= 0 && gpi == pj) || (gpj >= 0 && gpj == pi)) return 3;
    return 4;
}

// ---- warp / block reductions -------------------------------------------------
KF_DEV double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
KF_DEV long long warp_sum_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
KF_DEV double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic block sum (fixed tree for a fixed blockDim); scratch >= 32 doubles.
KF_DEV double block_sum(double v, double *scratch) {
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (wid == 0) {
        r = lane < nw ? scratch[lane] : 0.0;
        r = warp_sum(r);
        if (lane == 0) scratch[0] = r;
    }
    __syncthreads();
    r = scratch[0];
    __syncthreads();
    return r;
}
KF_DEV double block_max(double v, double *scratch) {
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (wid == 0) {
        r = lane < nw ? scratch[lane] : 0.0;
        r = warp_max(r);
        if (lane == 0) scratch[0] = r;
    }
    __syncthreads();
    r = scratch[0];
    __syncthreads();
    return r;
}

// ---- error plumbing (host) ---------------------------------------------------
void kf_set_error(const char *where, cudaError_t e);
// Every kernel launch of the library goes through this check, which also
// counts it (kf_launch_counter: the bench's gpu_launches).
void kf_count_launch();
#define KF_LAUNCH_CHECK(where)                                   \
    do {                                                         \
        kf_count_launch();                                       \
        cudaError_t _e = cudaGetLastError();                     \
        if (_e != cudaSuccess) { kf_set_error(where, _e); return 1; } \
    } while (0)
#define KF_CUDA(call, where)                                     \
    do {                                                         \
        cudaError_t _e = (call);                                 \
        if (_e != cudaSuccess) { kf_set_error(where, _e); return 1; } \
    } while (0)

static inline unsigned kf_blocks(long long n, int tpb) {
    return (unsigned)((n + tpb - 1) / tpb);
}
