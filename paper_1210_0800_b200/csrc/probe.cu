// probe.cu -- the FP64 roofline denominator, measured live on the device the
// bench runs on: throughput of independent DADD / DFMA chains over every SM
// (8 CTAs x 256 threads per SM, 8 independent chains per thread).
// MEASURED_PEAKS.json carries no FP64 figure; bench.py calls this before its
// timed region and reports the best of three launches.
#include <cuda_runtime.h>

#include "xqr_internal.h"

namespace {

template <int OP>
__global__ void __launch_bounds__(256) fp64_tput(double* out, int iters, double s) {
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = OP == 0 ? __dadd_rn(a[i], s) : __fma_rn(a[i], s, 1e-12);
    }
    double acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += a[i];
    if (acc == 12345.678) out[0] = acc;  // keeps the chains alive
}

}  // namespace

extern "C" int xqr_fp64_peak(xqr_ctx* ctx, int op, double* lane_instr_per_s) {
    if (!ctx || !lane_instr_per_s || (op != 0 && op != 1)) return XQR_USAGE;
    void* stream = xqr_ctx_stream(ctx);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return XQR_CUDA;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000, blocks = 8 * sms, threads = 256;
    double best = 0.0;
    for (int rep = 0; rep < 4; ++rep) {  // the first launch warms the clocks
        cudaEventRecord(e0, s);
        if (op == 0)
            fp64_tput<0><<<blocks, threads, 0, s>>>(out, iters, 1e-300);
        else
            fp64_tput<1><<<blocks, threads, 0, s>>>(out, iters, 1.0000001);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double rate = (double)blocks * threads * iters * 8 / (ms * 1e-3);
        if (rep > 0 && rate > best) best = rate;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess) return XQR_CUDA;
    *lane_instr_per_s = best;
    return XQR_OK;
}
