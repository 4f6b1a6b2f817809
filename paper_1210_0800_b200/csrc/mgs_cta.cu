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

// One system: the warp-specialised lane-pair sweep (flow_back_substitute), a
// CTA of 512 threads with x and the Smith records in shared memory.
template <int L>
__global__ void __launch_bounds__(512, 1) flow_backsub_kernel(BackSubParams p) {
    extern __shared__ double xs[];
    __shared__ unsigned long long s_key;
    __shared__ int s_sync[2 + 32];
    const int n = p.n;
    if (threadIdx.x == 0) s_key = kNoError;
    __syncthreads();
    bool bad = flow_back_substitute<L>(n, p.r, p.y, xs, xs + (size_t)n * 2 * L, s_sync, &s_key, 0);
    if (!bad)
        for (int e = threadIdx.x; e < n * 2 * L; e += blockDim.x) p.x[e] = xs[e];
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long key = s_key;
        xqr_status st;
        st.system = 0;
        st.code = key == kNoError ? 0 : (int)(key & 15);
        st.column = 0;
        p.st[0] = st;
    }
}

template <int L>
static cudaError_t launch_bs(const BackSubParams& p, cudaStream_t s) {
    const size_t flow_smem = sizeof(double) * (size_t)p.n * (5 * L + 1);
    // (quad-double only: double-double steps are too short to gain from it)
    if (L == 4 && p.batch == 1 && flow_smem <= 200 * 1024) {
        auto kern = flow_backsub_kernel<L>;
        if (flow_smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)flow_smem);
            if (e != cudaSuccess) return e;
        }
        kern<<<1, 512, flow_smem, s>>>(p);
        return cudaGetLastError();
    }
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
