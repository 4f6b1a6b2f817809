// mgs_cta.cu -- dispatch for the CTA-per-system MGS kernels (xmgs.cuh) and
// the standalone back-substitution kernel.
#include "xmgs.cuh"

namespace xb {

cudaError_t launch_mgs_L1_qr(const SolveParams&, cudaStream_t);
cudaError_t launch_mgs_L1_ls(const SolveParams&, cudaStream_t);
cudaError_t launch_mgs_L2_qr(const SolveParams&, cudaStream_t);
cudaError_t launch_mgs_L2_ls(const SolveParams&, cudaStream_t);
cudaError_t launch_mgs_L4_qr(const SolveParams&, cudaStream_t);
cudaError_t launch_mgs_L4_ls(const SolveParams&, cudaStream_t);

cudaError_t launch_mgs_cta(int limbs, bool lsq, const SolveParams& p, cudaStream_t s) {
    switch (limbs) {
        case 1: return lsq ? launch_mgs_L1_ls(p, s) : launch_mgs_L1_qr(p, s);
        case 2: return lsq ? launch_mgs_L2_ls(p, s) : launch_mgs_L2_qr(p, s);
        case 4: return lsq ? launch_mgs_L4_ls(p, s) : launch_mgs_L4_qr(p, s);
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
