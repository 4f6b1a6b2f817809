// mgs_grid_L4bs.cu -- instantiation unit for the single-system quad-double
// back substitution (grid2_backsub_kernel, xgrid2.cuh): its own unit so the
// CTA width (XB_G2BS_THREADS, and the merge slots sized to it) does not touch
// the grid kernels' shared memory.
#include "xgrid2.cuh"

namespace xb {
cudaError_t launch_grid_L4_backsub(const GridParams& p, cudaStream_t s) { return launch_grid2_backsub<4>(p, s); }
}  // namespace xb
