// coltask_bench.cu -- dev microbenchmark: throughput of the batched kernel's
// column task (remove_projection of one cqd 128-row column, xpair.cuh /
// xcolumn.cuh primitives) with no round structure around it: every warp of
// 2 CTAs x 8 warps per SM repeats tasks on its own column against rotating
// pivot columns in shared memory.  Prints column tasks/s and the FP64 issue
// fraction implied by the reference's work per task (8 leaf cmul + 7 in-lane
// and tree cadds ... = W_task below).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -DXB_CALLS=23 \
//        -I paper_1210_0800_b200/csrc tools/coltask_bench.cu -o tools/coltask_bench
#include <cstdio>

#include "xmgs.cuh"

using namespace xb;

constexpr int NW = 8, M = 128, NQ = 4;

__device__ unsigned long long mix(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ double urand(unsigned long long& s) {
    s = mix(s);
    return (double)(s >> 11) * 0x1p-53 - 0.5;
}
__device__ r4 rq(unsigned long long& s, double scale) {
    r4 v;
    v.c0 = scale * (1.0 + urand(s));
    v.c1 = v.c0 * 0x1p-54 * urand(s);
    v.c2 = v.c1 * 0x1p-54 * urand(s);
    v.c3 = v.c2 * 0x1p-54 * urand(s);
    renorm4(v.c0, v.c1, v.c2, v.c3);
    return v;
}

template <class W>
__global__ void __launch_bounds__(NW * 32, 2) bench(double* ws, int reps, int rpl, double* sink) {
    using F = typename W::F;
    const F f(rpl);
    extern __shared__ double smem[];  // NQ pivot columns
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long s = blockIdx.x * 7919ull + threadIdx.x * 104729ull + 1;
    // pivots: unit-ish columns (entries ~ 1/sqrt(m)); the task column ~ 1
    for (int e = threadIdx.x; e < NQ * f.COL; e += blockDim.x) {
        const int l = (e / f.LD) % 4;
        smem[e] = l == 0 ? 0.088 * (1.0 + urand(s)) : 0.088 * 0x1p-54 * urand(s) * (l == 1 ? 1 : 0x1p-54);
    }
    double* col = ws + ((size_t)blockIdx.x * NW + warp) * f.COL;
    for (int e = lane; e < f.COL; e += 32) {
        const int l = (e / f.LD) % 4;
        col[e] = l == 0 ? (1.0 + urand(s)) : 0x1p-54 * urand(s) * (l == 1 ? 1 : 0x1p-54);
    }
    __syncthreads();
    cx<r4> acc{};
    for (int r = 0; r < reps; ++r) {
        cx<r4> rr;
        W::remove_projection(f, smem + (r % NQ) * f.COL, col, lane, M, rr);
        if (lane == 0) acc.re.c0 += rr.re.c0;
    }
    if (lane == 0) sink[blockIdx.x * NW + warp] = acc.re.c0;
}

template <class W>
void run(const char* name, int rpl, int reps) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = 2 * sms;
    const size_t colb = sizeof(double) * 8 * 32 * 4;  // >= COL doubles for both formats
    double *ws, *sink;
    cudaMalloc(&ws, colb * blocks * NW);
    cudaMalloc(&sink, sizeof(double) * blocks * NW);
    const size_t smem = NQ * colb;
    cudaFuncSetAttribute(bench<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    bench<W><<<blocks, NW * 32, smem>>>(ws, 4, rpl, sink);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench<W><<<blocks, NW * 32, smem>>>(ws, reps, rpl, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // reference work per task (SURVEY Appendix B weights): m leaf cmul + (m-1)
    // cadd + m cmul + m csub (csub = cadd)
    const double w_task = M * 896.0 + (M - 1) * 180.0 + M * 896.0 + M * 180.0;
    const double tasks = (double)blocks * NW * reps;
    printf("%-10s %8.3f ms  %.3e tasks/s  FP64 issue frac %.3f  (%s)\n", name, ms, tasks / (ms * 1e-3),
           tasks * w_task / (ms * 1e-3) / 1.85e13, cudaGetErrorString(cudaGetLastError()));
    cudaFree(ws);
    cudaFree(sink);
}

int main() {
    run<mgs_pair<4>>("pair", 8, 200);
    run<mgs_warp<4, 3>>("warp", 4, 200);
    return 0;
}
