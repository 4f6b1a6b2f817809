// mgs_grid_L4.cu -- instantiation unit for the single-system cluster grid kernel (xgrid2.cuh).
#include "xgrid2.cuh"

namespace xb {
cudaError_t launch_grid_L4(const GridParams& p, int max_clusters, bool lsq, cudaStream_t s) {
    return launch_grid2<4>(p, lsq, max_clusters, s);
}
}  // namespace xb
