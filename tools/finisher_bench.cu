// finisher_bench.cu -- the back-substitution finisher step (update of x_{k-1} by
// x_k, then the Smith division; xbacksub.cuh) chained on one lane pair in
// isolation, SM cycles per step (dev tool):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -DXB_CALLS=1 \
//        -DXB_USE_SELP=1 -DXB_SHIFT_TAIL=1 -I paper_1210_0800_b200/csrc tools/finisher_bench.cu -o tools/fb_c1
#include <cstdio>
#include "xcolumn.cuh"
using namespace xb;
// one warp, lanes 0/1 = re/im halves: x_{k-1} = Smith((acc - r*x_k) / d), chained
__global__ void chain(const double* in, double* out, int steps, long long* cyc) {
    const int lane = threadIdx.x, part = lane & 1;
    if (lane >= 2) return;
    r4 v{in[part * 4 + 0], in[part * 4 + 1], in[part * 4 + 2], in[part * 4 + 3]};
    r4 rre{in[8], in[9], in[10], in[11]}, rim{in[12], in[13], in[14], in[15]};
    r4 acc{in[16 + part * 4], in[17 + part * 4], in[18 + part * 4], in[19 + part * 4]};
    r4 t{in[24], in[25], in[26], in[27]}, d{in[28], in[29], in[30], in[31]};
    int st = 0;
    recip_t<r4> rc = recip(d, st);
    long long c0 = clock64();
    for (int s = 0; s < steps; ++s) {
        const r4 y1 = v, y2 = shfl_pair(v, 3u);
        rpair<r4> pr = mul2(rre, y1, rim, y2);
        r4 u = sub(acc, add(pr.x, part ? pr.y : neg(pr.y)));
        const r4 ou = shfl_pair(u, 3u);
        const r4 are = part ? ou : u, aim = part ? u : ou;
        const r4 prod = mul(part ? are : aim, t);
        const r4 num = add(part ? aim : are, part ? neg(prod) : prod);
        v = divide_inline(num, d, rc);
    }
    long long c1 = clock64();
    out[lane * 4] = v.c0; out[lane * 4 + 1] = v.c1;
    if (lane == 0) *cyc = (c1 - c0) / steps;
}
int main() {
    double h[32];
    // full-limb values (renormalised on the device by construction below)
    double vals[8][2] = {{0.7, -0.3}, {0.2, -0.1}, {0.5, 0.25}, {0.37, 1.3}};
    auto put = [&](int o, double x) { h[o] = x; h[o + 1] = x * 0x1p-54 * 0.71; h[o + 2] = h[o + 1] * 0x1p-54 * -0.63; h[o + 3] = h[o + 2] * 0x1p-54 * 0.57; };
    put(0, 0.7); put(4, -0.3); put(8, 0.2); put(12, -0.1); put(16, 0.5); put(20, 0.25); put(24, 0.37); put(28, 1.3);
    (void)vals;
    double *din, *dout; long long* dc;
    cudaMalloc(&din, sizeof h); cudaMalloc(&dout, 64 * 8); cudaMalloc(&dc, 8);
    cudaMemcpy(din, h, sizeof h, cudaMemcpyHostToDevice);
    chain<<<1, 32>>>(din, dout, 64, dc);
    chain<<<1, 32>>>(din, dout, 256, dc);
    long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("finisher step (update + Smith) alone: %lld cycles\n", c);
}
