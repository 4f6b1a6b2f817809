// clusterbench.cu -- latency of cluster barriers and DSMEM loads on B200 (dev probe).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void __cluster_dims__(4, 1, 1) k_sync(int iters, long long* out) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) cg::this_cluster().sync();
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
}
__global__ void __cluster_dims__(4, 1, 1) k_dsmem(int iters, long long* out) {
    __shared__ double buf[64];
    buf[threadIdx.x % 64] = threadIdx.x;
    cg::this_cluster().sync();
    double* rem = cg::this_cluster().map_shared_rank(buf, (cg::this_cluster().block_rank() + 1) % 4);
    int idx = threadIdx.x % 64;
    double acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        double v = rem[idx];
        acc += v;
        idx = ((int)v + i) & 63;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (t1 - t0) / iters;
    if (acc == -1) out[2] = 1;
    cg::this_cluster().sync();
}
__global__ void k_bar(int iters, long long* out) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[3] = (t1 - t0) / iters;
}
int main() {
    long long* d;
    cudaMalloc(&d, 64);
    long long h[4];
    k_sync<<<4 * 37, 128>>>(1000, d);
    k_dsmem<<<4 * 37, 128>>>(1000, d);
    k_bar<<<148, 128>>>(1000, d);
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("cluster.sync (4 CTAs x 128 thr): %lld cycles\nDSMEM dependent load: %lld cycles\n__syncthreads (128 thr): %lld cycles\nerr=%s\n",
           h[0], h[1], h[3], cudaGetErrorString(cudaGetLastError()));
}
