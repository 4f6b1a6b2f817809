// FP64 pipe microbenchmark: throughput of independent DFMA/DADD chains and
// latency of one dependent DADD chain.  Used to set the FP64 roofline peak
// (MEASURED_PEAKS.json carries no FP64 figure).
#include <cstdio>
#include <cuda_runtime.h>

template <int OP, int ILP>
__global__ void tput(double* out, int iters, double s) {
    double a[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            if (OP == 0) a[i] = __fma_rn(a[i], s, 1e-12);
            else a[i] = __dadd_rn(a[i], s);
        }
    }
    double acc = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc += a[i];
    if (acc == 12345.678) out[0] = acc;
}

__global__ void lat(double* out, int iters, double s, long long* cyc) {
    double a = threadIdx.x;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        a = __dadd_rn(a, s); a = __dadd_rn(a, s); a = __dadd_rn(a, s); a = __dadd_rn(a, s);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = a; }
}

int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("name=%s sms=%d clock_khz=%d l2=%d smem_optin=%zu regs_per_sm=%d\n", p.name,
           p.multiProcessorCount, clk, p.l2CacheSize, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
    double* out; cudaMalloc(&out, 8);
    long long* cyc; cudaMalloc(&cyc, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 20000;
    for (int op = 0; op < 2; ++op) {
        for (int rep = 0; rep < 3; ++rep) {
            int blocks = p.multiProcessorCount * 8, threads = 256;
            cudaEventRecord(e0);
            if (op == 0) tput<0, 8><<<blocks, threads>>>(out, iters, 1.0000001);
            else tput<1, 8><<<blocks, threads>>>(out, iters, 1e-300);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double inst = (double)blocks * threads * iters * 8;
            printf("%s lane-instr/s = %.3e  (%.2f TFLOP/s fma=2)  ms=%.2f\n", op == 0 ? "DFMA" : "DADD",
                   inst / (ms * 1e-3), inst * (op == 0 ? 2 : 1) / (ms * 1e-3) / 1e12, ms);
        }
    }
    lat<<<1, 32>>>(out, 10000, 1e-300, cyc);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dependent DADD latency = %.2f cycles\n", (double)c / 40000.0);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
