// mgs_L2_qr.cu -- instantiation unit (see xmgs_launch.cuh).
#include "xmgs_launch.cuh"

namespace xb {
cudaError_t launch_mgs_L2_qr(const SolveParams& p, cudaStream_t s) { return launch_rpl<2, false>(p, s); }
}  // namespace xb
