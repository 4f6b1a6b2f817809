// mgs_L1_qr.cu -- instantiation unit (see xmgs_launch.cuh).
#include "xmgs_launch.cuh"

namespace xb {
cudaError_t launch_mgs_L1_qr(const SolveParams& p, cudaStream_t s) { return launch_rpl<1, false>(p, s); }
}  // namespace xb
