// mgs_cta.cu -- launchers for the CTA-per-system MGS kernels (xmgs.cuh).
#include "xmgs.cuh"

namespace xb {

// ---- launchers ----------------------------------------------------------------
constexpr int kWarps = 4;

// Minimum resident CTAs per SM requested from ptxas (caps registers).
template <int L, int LV>
constexpr int min_blocks() {
    return L == 4 ? (LV <= 3 ? 3 : 1) : (LV <= 3 ? 4 : 2);
}

template <int L, int LV, bool LSQ>
static cudaError_t launch_one(const SolveParams& p, int rpl, cudaStream_t s) {
    auto kern = mgs_cta_kernel<L, LV, kWarps, LSQ, min_blocks<L, LV>()>;
    const size_t smem = 2 * sizeof(double) * (size_t)(2 * L * 32 * rpl);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    kern<<<(unsigned)p.batch, kWarps * 32, smem, s>>>(p, rpl);
    return cudaGetLastError();
}

// Stack depth 3 serves m <= 128 (the batched hot path) with the fewest
// registers; depth 6 serves m <= 1024.
template <int L, bool LSQ>
static cudaError_t launch_rpl(const SolveParams& p, cudaStream_t s) {
    const int rpl = rows_per_lane(p.m);
    if (rpl <= 4) return launch_one<L, 3, LSQ>(p, rpl, s);
    if (rpl <= kMaxRowsPerLane) return launch_one<L, 6, LSQ>(p, rpl, s);
    return cudaErrorInvalidValue;
}

cudaError_t launch_mgs_cta(int limbs, bool lsq, const SolveParams& p, cudaStream_t s) {
    switch (limbs) {
        case 1: return lsq ? launch_rpl<1, true>(p, s) : launch_rpl<1, false>(p, s);
        case 2: return lsq ? launch_rpl<2, true>(p, s) : launch_rpl<2, false>(p, s);
        case 4: return lsq ? launch_rpl<4, true>(p, s) : launch_rpl<4, false>(p, s);
        default: return cudaErrorInvalidValue;
    }
}

template <int L>
static cudaError_t launch_bs(const BackSubParams& p, cudaStream_t s) {
    const size_t smem = sizeof(double) * (size_t)p.n * 2 * L;
    auto kern = back_substitute_kernel<L>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    kern<<<(unsigned)p.batch, 256, smem, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_back_substitute(int limbs, const BackSubParams& p, cudaStream_t s) {
    switch (limbs) {
        case 1: return launch_bs<1>(p, s);
        case 2: return launch_bs<2>(p, s);
        case 4: return launch_bs<4>(p, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace xb
