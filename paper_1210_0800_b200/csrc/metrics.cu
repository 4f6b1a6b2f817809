// metrics.cu -- the reference's verification metrics on the device
// (SURVEY.md §8f-1), batched over systems:
//   residual_max_entry   mgs.hpp:161-178  max |a_ij - sum_{l<=j} q_il r_lj|,
//                        the sum accumulated left to right in working precision;
//   orthogonality_defect mgs.hpp:208-222  max |(q_i^H q_j) - delta_ij| over
//                        i <= j, the inner product on the fixed tree
//                        (reduction.hpp:45-51).
// |z| is cabs = sqrt(re*re + im*im) (complex.hpp:77-85).  The maximum is
// order-independent, so the per-thread / per-block maxima combine in any
// order and the result is bitwise the reference's.  A non-finite value
// reports overflow (the reference's checked ops throw overflow_error).
#include "xbacksub.cuh"
#include "xcolumn.cuh"
#include "xqr_internal.h"

namespace xb {

template <int L>
XB_DEVICE real_t<L> cabs_ref(const cx<real_t<L>>& z) {
    rpair<real_t<L>> p = mul2(z.re, z.re, z.im, z.im);
    return rsqrt_ref(add(p.x, p.y));
}

// running maximum, reference comparison (`if (e > worst) worst = e`)
template <int L>
XB_DEVICE void keep_max(real_t<L>& worst, const real_t<L>& e) {
    if (lt(worst, e)) worst = e;
}

// block max of one value per thread into out[block] (L doubles); flags overflow
template <int L>
XB_DEVICE void block_max(real_t<L> v, bool bad, double* out, int* flag) {
    using R = real_t<L>;
    __shared__ double red[32 * 4];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        R other = shfl_down_r(v, o);
        if (lt(v, other)) v = other;
    }
    if (lane == 0) store_real<L>(red + warp * L, 1, v);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
    if (threadIdx.x == 0) {
        R best;
        load_real<L>(red, 1, best);
        for (int w = 1; w < nw; ++w) {
            R o;
            load_real<L>(red + w * L, 1, o);
            if (lt(best, o)) best = o;
        }
        store_real<L>(out, 1, best);
    }
}

// one thread per entry (i, j) of one system; grid (ceil(m*n/256), batch)
template <int L>
__global__ void __launch_bounds__(256) residual_kernel(int m, int n, const double* a, const double* q,
                                                       const double* r, double* part, int* flags) {
    using R = real_t<L>;
    using C = cx<R>;
    constexpr int L2 = 2 * L;
    const int64_t sys = blockIdx.y;
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const double* A = a + sys * (int64_t)m * n * L2;
    const double* Q = q + sys * (int64_t)m * n * L2;
    const double* Rm = r + sys * (int64_t)n * n * L2;
    R worst = rmake<R>(0.0);
    bool bad = false;
    if (e < (int64_t)m * n) {
        const int i = (int)(e % m), j = (int)(e / m);
        C s{rmake<R>(0.0), rmake<R>(0.0)};
#pragma unroll 1
        for (int l = 0; l <= j; ++l)
            s = cadd(s, cmul(load_aos<L>(Q + ((int64_t)l * m + i) * L2), load_aos<L>(Rm + ((int64_t)j * n + l) * L2)));
        worst = cabs_ref<L>(csub(load_aos<L>(A + ((int64_t)j * m + i) * L2), s));
        bad = !vfinite(worst);
    }
    block_max<L>(worst, bad, part + (sys * gridDim.x + blockIdx.x) * L, flags + sys);
}

// one warp per pair (i, j), i <= j, of one system; grid (ceil(pairs/8), batch)
template <int L, int LV>
__global__ void __launch_bounds__(256) orthodefect_kernel(int m, int n, int rpl, const double* q,
                                                          double* part, int* flags) {
    using R = real_t<L>;
    using C = cx<R>;
    constexpr int L2 = 2 * L;
    const int64_t sys = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int64_t pid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t npairs = (int64_t)n * (n + 1) / 2;
    const double* Q = q + sys * (int64_t)m * n * L2;
    R worst = rmake<R>(0.0);
    bool bad = false;
    if (pid < npairs) {
        // pid -> (i, j) with i <= j, row-major over i
        int i = 0;
        int64_t rem = pid;
        while (rem >= n - i) {
            rem -= n - i;
            ++i;
        }
        const int j = i + (int)rem;
        const double* qi = Q + (int64_t)i * m * L2;
        const double* qj = Q + (int64_t)j * m * L2;
        int cnt = m - lane * rpl;
        cnt = cnt < 0 ? 0 : (cnt > rpl ? rpl : cnt);
        C acc = lane_tree<LV, C>(cnt, [&](int t) {
            const int row = lane * rpl + t;
            return cmul(cconj(load_aos<L>(qi + (int64_t)row * L2)), load_aos<L>(qj + (int64_t)row * L2));
        });
        acc = warp_tree(acc, lane, m, rpl);
        if (i == j) acc.re = sub(acc.re, rmake<R>(1.0));
        worst = cabs_ref<L>(acc);
        bad = !vfinite(worst);
        worst = shfl_idx_r(worst, 0);
        bad = __shfl_sync(0xffffffffu, (int)bad, 0) != 0;
    }
    block_max<L>(worst, bad, part + (sys * gridDim.x + blockIdx.x) * L, flags + sys);
}

// final max over the per-block partials of each system
template <int L>
__global__ void final_max_kernel(int nblocks, const double* part, double* out, const int* flags,
                                 xqr_status* st) {
    using R = real_t<L>;
    const int64_t sys = blockIdx.x;
    if (threadIdx.x == 0 && st) {
        xqr_status v;
        v.code = flags[sys] ? XQR_OVERFLOW : XQR_OK;
        v.column = 0;
        v.system = sys;
        st[sys] = v;
    }
    R best = rmake<R>(0.0);
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
        R v;
        load_real<L>(part + (sys * nblocks + b) * L, 1, v);
        if (lt(best, v)) best = v;
    }
    block_max<L>(best, false, out + sys * L, nullptr);
}

template <int L>
cudaError_t launch_metric_t(int which, int64_t batch, int m, int n, const double* a, const double* q,
                            const double* r, double* out, double* part, int* flags, xqr_status* st,
                            cudaStream_t s) {
    int nblocks;
    if (which == 0) {
        nblocks = (int)(((int64_t)m * n + 255) / 256);
        residual_kernel<L><<<dim3(nblocks, (unsigned)batch), 256, 0, s>>>(m, n, a, q, r, part, flags);
    } else {
        const int64_t npairs = (int64_t)n * (n + 1) / 2;
        nblocks = (int)((npairs + 7) / 8);
        const int rpl = rows_per_lane(m);
        // in-lane tree depth: the binary counter holds up to 2^LV - 1 leaves
        if (rpl <= 4)
            orthodefect_kernel<L, 3><<<dim3(nblocks, (unsigned)batch), 256, 0, s>>>(m, n, rpl, q, part, flags);
        else if (rpl <= 32)
            orthodefect_kernel<L, 6><<<dim3(nblocks, (unsigned)batch), 256, 0, s>>>(m, n, rpl, q, part, flags);
        else
            orthodefect_kernel<L, 7><<<dim3(nblocks, (unsigned)batch), 256, 0, s>>>(m, n, rpl, q, part, flags);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    final_max_kernel<L><<<(unsigned)batch, 128, 0, s>>>(nblocks, part, out, flags, st);
    return cudaGetLastError();
}

// scratch: partial maxima, batch * metric_blocks(...) * L doubles
int64_t metric_blocks(int which, int m, int n) {
    return which == 0 ? ((int64_t)m * n + 255) / 256 : ((int64_t)n * (n + 1) / 2 + 7) / 8;
}

cudaError_t launch_metric(int limbs, int which, int64_t batch, int m, int n, const double* a,
                          const double* q, const double* r, double* out, double* part, int* flags,
                          xqr_status* st, cudaStream_t s) {
    switch (limbs) {
        case 1: return launch_metric_t<1>(which, batch, m, n, a, q, r, out, part, flags, st, s);
        case 2: return launch_metric_t<2>(which, batch, m, n, a, q, r, out, part, flags, st, s);
        case 4: return launch_metric_t<4>(which, batch, m, n, a, q, r, out, part, flags, st, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace xb
