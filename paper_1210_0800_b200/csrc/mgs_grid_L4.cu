// mgs_grid_L4.cu -- instantiation unit for the single-system cluster grid
// kernel (xgrid2.cuh), one row per lane pair (m <= 256), and the launch
// entry point with the back substitution.  Wider rows: mgs_grid_L4w.cu.
#include "xgrid2.cuh"

namespace xb {
cudaError_t launch_grid_L4_wide(const GridParams& p, int max_clusters, bool lsq, cudaStream_t s);
cudaError_t launch_grid_L4_backsub(const GridParams& p, cudaStream_t s);

cudaError_t launch_grid_L4(const GridParams& p, int max_clusters, bool lsq, cudaStream_t s) {
    cudaError_t e;
    switch (p.rpt) {
        case 1: e = launch_grid2_rpp<4, 1>(p, lsq, max_clusters, s); break;
        case 2:
        case 4: e = launch_grid_L4_wide(p, max_clusters, lsq, s); break;
        default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess || !lsq) return e;
    return launch_grid_L4_backsub(p, s);
}
}  // namespace xb
