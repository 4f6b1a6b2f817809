// mgs_L2_ls.cu -- instantiation unit (see xmgs_launch.cuh).
#include "xmgs_launch.cuh"

namespace xb {
cudaError_t launch_mgs_L2_ls(const SolveParams& p, cudaStream_t s) { return launch_rpl<2, true>(p, s); }
}  // namespace xb
