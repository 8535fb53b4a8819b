// FMA issue-rate microbenchmarks: the FP32 / FP64 denominators of the pair
// and solvation kernels' rooflines (MEASURED_PEAKS.json carries only HBM and
// bf16 tensor figures).  Each thread runs 8 independent FMA chains.
#include "kf_common.cuh"

namespace {
template <typename T>
__global__ void __launch_bounds__(256) fma_kernel(T *out, int iters, T a, T b) {
    T x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = (T)(threadIdx.x + k) * (T)1e-3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    T s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == (T)123.456) out[0] = s;   // keep the chains live
}
}  // namespace

extern "C" int kf_peak_flops(int kind, double *out, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0, sms = 0;
    KF_CUDA(cudaGetDevice(&dev), "get device");
    KF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
    const int blocks = sms * 8, threads = 256, iters = kind == 0 ? 4096 : 1024;
    void *buf = nullptr;
    KF_CUDA(cudaMallocAsync(&buf, 16, s), "peak buf");
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0, s);
        if (kind == 0) fma_kernel<float><<<blocks, threads, 0, s>>>((float *)buf, iters, 0.9999f, 1e-4f);
        else fma_kernel<double><<<blocks, threads, 0, s>>>((double *)buf, iters, 0.9999, 1e-4);
        cudaEventRecord(e1, s);
        KF_CUDA(cudaEventSynchronize(e1), "peak sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(buf, s);
    KF_LAUNCH_CHECK("fma_kernel");
    *out = 2.0 * 8.0 * (double)iters * blocks * threads / (best * 1e-3);
    return 0;
}
