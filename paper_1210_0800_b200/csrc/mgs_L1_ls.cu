// mgs_L1_ls.cu -- instantiation unit (see xmgs_launch.cuh).
#include "xmgs_launch.cuh"

namespace xb {
cudaError_t launch_mgs_L1_ls(const SolveParams& p, cudaStream_t s) { return launch_rpl<1, true>(p, s); }
}  // namespace xb
