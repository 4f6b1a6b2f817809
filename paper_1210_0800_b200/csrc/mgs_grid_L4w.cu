// mgs_grid_L4w.cu -- instantiation unit for the single-system cluster grid
// kernel (xgrid2.cuh) with 2 or 4 rows per lane pair (256 < m <= 1024).
#include "xgrid2.cuh"

namespace xb {
cudaError_t launch_grid_L4_wide(const GridParams& p, int max_clusters, bool lsq, cudaStream_t s) {
    return p.rpt == 2 ? launch_grid2_rpp<4, 2>(p, lsq, max_clusters, s)
                      : launch_grid2_rpp<4, 4>(p, lsq, max_clusters, s);
}
}  // namespace xb
