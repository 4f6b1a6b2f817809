// mgs_grid_L1.cu -- instantiation unit for the single-system grid kernel (xgrid1.cuh).
#include "xgrid1.cuh"

namespace xb {
cudaError_t launch_grid_L1(const GridParams& p, int grid, bool lsq, cudaStream_t s) {
    return lsq ? launch_grid1<1, true>(p, grid, s) : launch_grid1<1, false>(p, grid, s);
}
}  // namespace xb
