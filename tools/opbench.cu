// opbench.cu -- throughput of the device dd/qd operations (xarith.cuh) on a
// full GPU: every thread runs NCH independent dependency chains of K ops on
// per-lane random operands (lanes diverge exactly as in the batched solver).
// Prints ns per op per SM and the FP64 issue fraction implied by the
// reference's per-op instruction weights.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 \
//        -I paper_1210_0800_b200/csrc tools/opbench.cu -o tools/opbench
#include <cstdio>
#include <cstdlib>

#include "xarith.cuh"

using namespace xb;

constexpr int K = 64;

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ double urand(unsigned long long& s) {
    s = mix(s);
    return (double)(s >> 11) * 0x1p-53;
}
__device__ r4 rq(unsigned long long& s, int e) {
    r4 v;
    v.c0 = ldexp(1.0 + urand(s), e) * (urand(s) < 0.5 ? -1.0 : 1.0);
    v.c1 = v.c0 * 0x1p-54 * (2 * urand(s) - 1);
    v.c2 = v.c1 * 0x1p-54 * (2 * urand(s) - 1);
    v.c3 = v.c2 * 0x1p-54 * (2 * urand(s) - 1);
    renorm4(v.c0, v.c1, v.c2, v.c3);
    return v;
}
__device__ r2 rd(unsigned long long& s, int e) {
    r2 v;
    v.c0 = ldexp(1.0 + urand(s), e) * (urand(s) < 0.5 ? -1.0 : 1.0);
    v.c1 = v.c0 * 0x1p-54 * (2 * urand(s) - 1);
    double t = v.c0;
    v.c0 = t + v.c1;
    v.c1 = v.c1 - (v.c0 - t);
    return v;
}

template <class R>
__device__ R rr(unsigned long long& s, int e);
template <>
__device__ r4 rr<r4>(unsigned long long& s, int e) { return rq(s, e); }
template <>
__device__ r2 rr<r2>(unsigned long long& s, int e) { return rd(s, e); }

// op 0: add  x = (x + y_t) - y'_t-ish (bounded): x = add(x, y[t&3]); y's alternate sign
// op 1: mul  x = x * y[t&3] with |y| ~ 1
// op 2: cmul
// op 3: cadd
// op 4: axpy a = a - r*q (the MGS update)
template <class R, int OP, int NCH>
__global__ void __launch_bounds__(128) bench(double* sink, int reps) {
    unsigned long long s = blockIdx.x * 1315423911ull + threadIdx.x * 2654435761ull + 7;
    cx<R> x[NCH], y[4];
#pragma unroll
    for (int c = 0; c < NCH; ++c) x[c] = {rr<R>(s, 0), rr<R>(s, 0)};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        y[t] = {rr<R>(s, 0), rr<R>(s, 0)};
    }
    for (int r = 0; r < reps; ++r) {
#pragma unroll 1
        for (int t = 0; t < K; ++t) {
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                const cx<R>& w = y[(t + c) & 3];
                if (OP == 0) x[c].re = add(x[c].re, (t & 1) ? neg(w.re) : w.re);
                if (OP == 1) x[c].re = mul(x[c].re, w.re);
                if (OP == 2) x[c] = cmul(x[c], w);
                if (OP == 3) x[c] = cadd(x[c], (t & 1) ? cx<R>{neg(w.re), neg(w.im)} : w);
                if (OP == 4) x[c] = csub(x[c], cmul(w, y[(t + c + 1) & 3]));
                // zero-limb operands (widened constants): the general paths
                if (OP == 5) x[c].re = add(x[c].re, rmake<R>((t & 1) ? -1.0 : 1.0));
                if (OP == 6) x[c].re = mul(x[c].re, rmake<R>((t & 1) ? 0.75 : 1.3125));
            }
        }
    }
    double acc = 0;
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc += head(x[c].re) + head(x[c].im);
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <class R, int OP, int NCH>
void run(const char* name, double fp64_per_op, int blocks_per_sm, int sms, double* sink) {
    const int blocks = blocks_per_sm * sms, reps = 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    bench<R, OP, NCH><<<blocks, 128>>>(sink, 1);
    cudaEventRecord(e0);
    bench<R, OP, NCH><<<blocks, 128>>>(sink, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * 128 * NCH * K * reps;
    const double rate = ops / (ms * 1e-3);
    const double instr = rate * fp64_per_op;
    printf("%-10s nch=%d blk/SM=%d  %8.3f ms  %.3e op/s  FP64 instr/s %.3e (%.1f%% of 1.85e13)  err=%s\n",
           name, NCH, blocks_per_sm, ms, rate, instr, 100 * instr / 1.85e13,
           cudaGetErrorString(cudaGetLastError()));
}

// latency: one warp, one dependent chain; ns per op
template <class R, int OP>
void lat(const char* name, double* sink, int blocks = 1, int threads = 32) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    bench<R, OP, 1><<<blocks, threads>>>(sink, 1);
    cudaEventRecord(e0);
    bench<R, OP, 1><<<blocks, threads>>>(sink, 16);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ns = ms * 1e6 / (16.0 * K);
    printf("latency %-10s %4dx%-4d %8.1f ns/op  (%6.0f cycles at 1.965 GHz)\n", name, blocks, threads, ns, ns * 1.965);
}

int main() {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* sink;
    cudaMalloc(&sink, sizeof(double) * 148 * 64 * 128);
    // reference per-op FP64 instruction weights (Appendix B): qd add 90, mul 179,
    // cmul 896, cadd 180; dd add 20, mul 9, cmul 76, cadd 40
    lat<r4, 0>("qd add", sink);
    lat<r4, 0>("qd add", sink, 1, 128);
    lat<r4, 0>("qd add", sink, 148, 128);
    lat<r4, 0>("qd add", sink, 148, 64);
    lat<r4, 1>("qd mul", sink, 148, 128);
    lat<r4, 1>("qd mul", sink);
    lat<r4, 2>("qd cmul", sink);
    lat<r4, 3>("qd cadd", sink);
    lat<r4, 4>("qd axpy", sink);
    lat<r4, 5>("qd add0", sink);
    lat<r4, 6>("qd mul0", sink);
    lat<r2, 0>("dd add", sink);
    lat<r2, 1>("dd mul", sink);
    for (int bps : {4, 8}) {
        run<r4, 0, 1>("qd add", 90, bps, sms, sink);
        run<r4, 0, 2>("qd add", 90, bps, sms, sink);
        run<r4, 1, 1>("qd mul", 179, bps, sms, sink);
        run<r4, 1, 2>("qd mul", 179, bps, sms, sink);
        run<r4, 2, 1>("qd cmul", 896, bps, sms, sink);
        run<r4, 3, 1>("qd cadd", 180, bps, sms, sink);
        run<r4, 4, 1>("qd axpy", 1076, bps, sms, sink);
        run<r2, 2, 1>("dd cmul", 76, bps, sms, sink);
        run<r2, 3, 1>("dd cadd", 40, bps, sms, sink);
        run<r2, 4, 1>("dd axpy", 116, bps, sms, sink);
    }
    return 0;
}
