// xqr_internal.h -- launch interface between the C ABI (capi.cu) and the
// kernels (mgs_cta.cu, arith.cu).  Not part of the public boundary.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/xqr_b200.h"

namespace xb {

// Status key: the first error in the reference's program order wins
// (atomicMin).  pos enumerates program points:
//   0                      norm pre-pass (mgs.hpp:91-96 / :143)
//   1 + k*(C+1)            normalize column k       (mgs.hpp:99 / :149)
//   1 + k*(C+1) + (j-k)    remove_projection(k, j)   (mgs.hpp:101-103 / :150-153)
//   1 + n*(C+1)            z = column_norm(b)        (mgs.hpp:155)
//   2 + n*(C+1) + (n-1-k)  back substitution step k  (mgs.hpp:117-124)
// with C = number of factored columns (n for QR, n+1 for LS).
__host__ __device__ inline unsigned long long status_key(long long pos, int column, int code) {
    return ((unsigned long long)pos << 24) | ((unsigned long long)(column & 0xFFFFF) << 4) |
           (unsigned long long)code;
}
constexpr unsigned long long kNoError = ~0ull;

struct SolveParams {
    int64_t batch;
    int m, n;
    const double* a;  // AoS, batch * m*n*2L
    const double* b;  // AoS, batch * m*2L (LS only)
    double* q;        // AoS out (QR only)
    double* r;        // AoS out n x n (QR only)
    double* x;        // AoS out n (LS only)
    double* z;        // L doubles per system (LS only)
    xqr_status* st;   // per system
    double* ws;       // lane-interleaved planar columns, ws_stride doubles per system
    int64_t ws_stride;
    double* rws;      // LS: R (n*n*2L) + y (n*2L) + Smith prep (n*(3L+1)) per system
    int64_t rws_stride;
};

// rows-per-lane for a one-warp-per-column task
inline int rows_per_lane(int m) {
    int r = 1;
    while (32 * r < m) r <<= 1;
    return r;
}
constexpr int kMaxRowsPerLane = 32;  // m <= 1024
// rows per lane PAIR (16 pairs per warp, xpair.cuh): quad-double m <= 128
inline int rows_per_pair(int m) {
    int r = 1;
    while (16 * r < m) r <<= 1;
    return r;
}


// doubles of planar workspace per system (32 x rows per lane per column;
// also covers the lane-pair layout: 16 x rows_per_pair(m) <= 32 x rows_per_lane(m))
inline int64_t ws_doubles(int limbs, int m, int ncols) {
    return (int64_t)ncols * 2 * limbs * 32 * rows_per_lane(m);
}
inline int64_t rws_doubles(int limbs, int n) {
    return (int64_t)n * n * 2 * limbs + (int64_t)n * 2 * limbs + (int64_t)n * (3 * limbs + 1);
}

cudaError_t launch_mgs_cta(int limbs, bool lsq, const SolveParams& p, cudaStream_t s);

struct BackSubParams {
    int64_t batch;
    int n;
    const double* r;  // AoS n x n per system
    const double* y;  // AoS n per system
    double* x;        // AoS n per system
    xqr_status* st;
    double* prep;     // n*(3L+1) per system
};
cudaError_t launch_back_substitute(int limbs, const BackSubParams& p, cudaStream_t s);

// Single-system cluster grid kernel (xgrid2.cuh): a column per cluster of
// `cs` CTAs of 128 threads, a lane pair per row (rpt = rows per lane pair).
struct GridParams {
    int m, n;
    int rpt;            // xgrid2: rows per lane pair (1 or 2); xgrid1: rows per thread
    const double* a;    // AoS m x n
    const double* b;    // AoS m (LS)
    double* q;          // AoS out (QR)
    double* r;          // AoS out n x n (QR)
    double* x;          // AoS out n (LS)
    double* z;          // L doubles (LS)
    xqr_status* st;
    double* ws;         // xgrid2: AoS working copy (ncol * m * 2L); xgrid1: planar columns
    double* rws;        // LS: R (n*n*2L) + y (n*2L) + Smith prep (n*(3L+1))
    double* norms;      // ncol * L
    int* flags;         // n: arrivals of the owner cluster's CTAs
    unsigned long long* key;    // global status key (init kNoError)
    unsigned long long* trace;  // optional (dev): 4 globaltimer stamps per pivot
    int cs;                     // CTAs per cluster
    int* counters;              // [0] pre-pass arrivals, [1] final arrivals, [2] abort word
    int pair_bulk;              // xgrid2: update trailing columns two at a time (lockstep)
    int chain;                  // xgrid1: CTA 0 runs every pivot (chain mode, xgrid1.cuh)
    int* cflags;                // xgrid1 chain mode, ncol: projections applied per column
    int64_t sys;                // index written into the status (a batch solved system by system)
};

// single systems (the grid kernels) take m <= kGridMaxRows; batches (one CTA
// per system) m <= 32 * kMaxRowsPerLane
constexpr int kGridMaxRows = 2048;
// quad-double (xgrid2.cuh): CTAs per cluster, rows per lane pair, and whether
// trailing columns are updated two at a time.  Two CTAs share each SM.
// Measured (tools/trace_single.py, same box): m <= 256 -> clusters of up to
// 4 CTAs, one row per lane pair; 256 < m <= 512 -> 8-CTA clusters, one row
// per lane pair, paired bulk updates (13.3 vs 14.1 ms for 4 CTAs x 2 rows:
// the shorter per-pivot chain wins once the bulk keeps up); m > 512 -> 4 CTAs.
constexpr int kGrid2PerSM = 2;
inline void grid_shape(int m, int& cs, int& rpp, int& pair) {
    if (m > 256 && m <= 512) {
        cs = 8;
        rpp = 1;
        pair = 1;
        return;
    }
    if (m > 1024) {  // up to kGridMaxRows = 2048: 8 CTAs x 64 lane pairs x 4 rows
        cs = 8;
        rpp = 4;
        pair = 0;
        return;
    }
    const int need = (m + 63) / 64;
    cs = 1;
    while (cs < need && cs < 4) cs <<= 1;
    rpp = 1;
    while (cs * 64 * rpp < m) rpp <<= 1;
    pair = 0;
}
// double / double-double (xgrid1.cuh): rows per thread of a 256-thread CTA
inline int grid1_rows_per_thread(int m) {
    int r = 1;
    while (256 * r < m) r <<= 1;
    return r;
}
cudaError_t launch_grid_L1(const GridParams& p, int grid, bool lsq, cudaStream_t s);
cudaError_t launch_grid_L2(const GridParams& p, int grid, bool lsq, cudaStream_t s);
cudaError_t launch_grid_L4(const GridParams& p, int max_clusters, bool lsq, cudaStream_t s);

// verification metrics (metrics.cu): which 0 = residual_max_entry, 1 = orthogonality_defect
int64_t metric_blocks(int which, int m, int n);
cudaError_t launch_metric(int limbs, int which, int64_t batch, int m, int n, const double* a,
                          const double* q, const double* r, double* out, double* part, int* flags,
                          xqr_status* st, cudaStream_t s);

cudaError_t launch_arith(int limbs, int op, int64_t count, const double* a, const double* b,
                         double* out, int32_t* codes, cudaStream_t s);

}  // namespace xb
