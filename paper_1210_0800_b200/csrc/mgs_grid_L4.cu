// mgs_grid_L4.cu -- instantiation unit for the single-system grid kernel (xgrid.cuh).
#include "xgrid.cuh"

namespace xb {
cudaError_t launch_grid_L4(const GridParams& p, int grid, bool lsq, cudaStream_t s) {
    return lsq ? launch_grid<4, true>(p, grid, s) : launch_grid<4, false>(p, grid, s);
}
}  // namespace xb
