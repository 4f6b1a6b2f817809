// mgs_L4_qr.cu -- instantiation unit (see xmgs_launch.cuh).
#include "xmgs_launch.cuh"

namespace xb {
cudaError_t launch_mgs_L4_qr(const SolveParams& p, cudaStream_t s) { return launch_rpl<4, false>(p, s); }
}  // namespace xb
