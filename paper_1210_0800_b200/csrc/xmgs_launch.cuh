// xmgs_launch.cuh -- launch templates for the CTA-per-system MGS kernels.
// Each (limbs, mode) pair is instantiated in its own translation unit
// (mgs_L*_*.cu) so the heavy quad-double kernels compile in parallel.
#pragma once
#include <atomic>
#include "xmgs.cuh"

namespace xb {

// Warps per CTA.  The quad-double m <= 128 kernel (the batched hot path)
// runs 8 warps x 2 CTAs per SM: the same 16 warps and 128 registers per
// thread as 4 x 4, but twice the columns of one system in flight, which
// hides more of the look-ahead normalisation and halves the last-wave tail
// (measured +2.2% systems/s on cqd 128x128, profiles/README.md).
#ifndef XB_CTA_WARPS4
#define XB_CTA_WARPS4 8
#endif
#ifndef XB_MINB4
#define XB_MINB4 2
#endif
template <int L, int LV>
constexpr int cta_warps() {
    return (L == 4 && LV <= 3) ? XB_CTA_WARPS4 : 4;
}

// Minimum resident CTAs per SM requested from ptxas (caps registers).
template <int L, int LV>
constexpr int min_blocks() {
    return L == 4 ? (LV <= 3 ? XB_MINB4 : 1) : (LV <= 3 ? 4 : 2);
}

// Opt a kernel in to `bytes` of dynamic shared memory; `allowed` (one per
// kernel instance, kept by the caller) remembers the largest size granted
// on each device (the attribute belongs to the device's context).
constexpr int kMaxDevices = 64;
template <class K>
static cudaError_t allow_dynamic_smem(K kern, size_t bytes, std::atomic<size_t>* allowed) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
    if (bytes <= allowed[dev].load(std::memory_order_relaxed)) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) {
        size_t cur = allowed[dev].load(std::memory_order_relaxed);
        while (cur < bytes && !allowed[dev].compare_exchange_weak(cur, bytes)) {
        }
    }
    return e;
}

template <int L, int LV, bool LSQ>
static cudaError_t launch_one(const SolveParams& p, int rpl, cudaStream_t s) {
    constexpr int NW = cta_warps<L, LV>();
#if XB_XSMEM
    static_assert(NW * 32 <= XB_XS_THREADS, "the qd add's shared-memory slots (xarith.cuh) cover every thread");
#endif
    auto kern = mgs_cta_kernel<mgs_warp<L, LV>, NW, LSQ, min_blocks<L, LV>()>;
    const size_t smem = 2 * sizeof(double) * (size_t)(2 * L * 32 * rpl);
    // static (the qd add's slots) + dynamic shared memory may exceed 48 KB
    static std::atomic<size_t> allowed[kMaxDevices];  // per template instance = per kernel
    if (cudaError_t e = allow_dynamic_smem(kern, smem, allowed)) return e;
    kern<<<(unsigned)p.batch, NW * 32, smem, s>>>(p, rpl);
    return cudaGetLastError();
}

// Lane-pair primitives (xpair.cuh) for quad-double m <= 128: rows per pair
// rpp = 16 pairs * rpp >= m.  12 warps x 2 CTAs per SM (80 registers, the
// caller-saved values around the qd calls spill): 24 warps hide more of the
// qd add's dependent-DADD latency than 16 warps at 128 registers -- measured
// on 4096 x cqd 128x128: 8 warps 4,520 sys/s, 12 4,621, 14 4,572, 16 4,353;
// 8 warps x 3 CTAs 4,610, 6 x 4 4,458, 8 x 4 4,236.
#ifndef XB_PAIR_WARPS
#define XB_PAIR_WARPS 12
#endif
#ifndef XB_PAIR_MINB
#define XB_PAIR_MINB 2
#endif
#ifndef XB_USE_PAIR
#define XB_USE_PAIR 1
#endif
template <int L, bool LSQ>
static cudaError_t launch_pair(const SolveParams& p, int rpp, cudaStream_t s) {
    constexpr int NW = XB_PAIR_WARPS;
#if XB_XSMEM
    static_assert(NW * 32 <= XB_XS_THREADS, "the qd add's shared-memory slots (xarith.cuh) cover every thread");
#endif
    auto kern = mgs_cta_kernel<mgs_pair<L>, NW, LSQ, XB_PAIR_MINB>;
    const size_t smem = 2 * sizeof(double) * (size_t)(2 * L * 16 * rpp);
    // static (the qd add's slots) + dynamic shared memory may exceed 48 KB
    static std::atomic<size_t> allowed[kMaxDevices];  // per template instance = per kernel
    if (cudaError_t e = allow_dynamic_smem(kern, smem, allowed)) return e;
    kern<<<(unsigned)p.batch, NW * 32, smem, s>>>(p, rpp);
    return cudaGetLastError();
}

// Stack depth 3 serves m <= 128 (the batched hot path) with the fewest
// registers; depth 6 serves m <= 1024.
template <int L, bool LSQ>
static cudaError_t launch_rpl(const SolveParams& p, cudaStream_t s) {
    if constexpr (L == 4 && XB_USE_PAIR)
        if (p.m <= 128) return launch_pair<L, LSQ>(p, rows_per_pair(p.m), s);
    const int rpl = rows_per_lane(p.m);
    if (rpl <= 4) return launch_one<L, 3, LSQ>(p, rpl, s);
    if (rpl <= kMaxRowsPerLane) return launch_one<L, 6, LSQ>(p, rpl, s);
    return cudaErrorInvalidValue;
}


}  // namespace xb
