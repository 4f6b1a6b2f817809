// mgs_grid_L1.cu -- instantiation unit for the single-system cluster grid kernel (xgrid2.cuh).
#include "xgrid2.cuh"

namespace xb {
cudaError_t launch_grid_L1(const GridParams& p, int max_clusters, bool lsq, cudaStream_t s) {
    return launch_grid2<1>(p, lsq, max_clusters, s);
}
}  // namespace xb
