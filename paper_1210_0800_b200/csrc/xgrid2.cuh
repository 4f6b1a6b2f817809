// xgrid2.cuh -- single-system MGS QR / least squares over the whole GPU,
// latency-first layout (configs 2-4: cdd/cqd 256x256, cqd 512x256).
//
// What bounds one large system is the per-pivot dependency chain
//   rp(k, k+1) -> |a_{k+1}|^2 tree -> sqrt -> reciprocal -> divide -> publish,
// and inside it the latency of one quad-double operation, which is set by the
// FP64 issue of ONE warp on its SM sub-partition (a warp FP64 instruction
// occupies the 16-lane pipe for 2 cycles).  So the layout minimises the
// quad-double work per lane on that chain:
//   * a LANE PAIR owns a row: the even lane computes the real part, the odd
//     lane the imaginary part of every complex quantity (the two halves of a
//     complex multiply / add / divide are independent -- complex.hpp:26-65);
//   * a column belongs to a thread-block CLUSTER of CS CTAs (grid_shape:
//     up to 4 for m <= 256, 8 for 256 < m <= 512 and m > 1024): 4 warps per
//     CTA, 16 lane pairs per warp; two CTAs (of different clusters) share an
//     SM, so one cluster's latency-bound chains fill the other's issue gaps;
//   * the fixed reduction tree (reduction.hpp:34-40) runs in-lane (rows of a
//     pair), then over lane pairs by shuffles, then over the cluster's warp
//     partials, staged into local shared memory with one DSMEM load per
//     thread -- the same pairing as the sequential tree_reduce, since rows
//     are laid out consecutively;
//   * warp 0 of each CTA computes the pivot's sqrt / reciprocal (call-form
//     qd ops: one hot copy in the instruction cache) and shares them through
//     shared memory, then each lane divides its own half of its row;
//   * for 256 < m <= 512 the trailing (off-chain) columns are updated two at
//     a time in lockstep (addc2, g2_tree2).
// Columns are distributed cyclically over clusters (column j -> cluster
// j mod G); q_k is the finished column itself in the (AoS) workspace,
// published with a release counter (carrying a failure bit) and acquired by
// every other cluster; the owner of column k+1 updates and normalises it
// first (look-ahead).  The
// working copy uses the reference's own memory image (column-major, row =
// re limbs then im limbs), so the loads of a lane pair are contiguous.
#pragma once
#include <cooperative_groups.h>
#include <cstdlib>

#include "xbacksub.cuh"
#include "xcolumn.cuh"
#include "xqr_internal.h"

namespace xb {

constexpr int kG2Threads = 128;
constexpr int kG2Warps = 4;
constexpr int kG2Pairs = 64;  // lane pairs (rows per step) per CTA

XB_DEVICE unsigned long long g2_timer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
XB_DEVICE int g2_ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
XB_DEVICE void g2_red_release(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// the warp of each CTA that runs a pivot's scalar chain (sqrt, reciprocal)
#ifndef XB_CHAIN_WARP
#define XB_CHAIN_WARP 0
#endif

template <int L, int RPP>
struct g2 {
    using R = real_t<L>;
    using C = cx<R>;
    static constexpr int L2 = 2 * L;

    int m, n, ncol, cs, crank, tid, lane, warp, part, pair, gpair, row0, cnt;
    double* ws;

    XB_DEVICE double* col(int j) const { return ws + (int64_t)j * m * L2; }
    // own half of row i of a column
    XB_DEVICE R ld_part(const double* c, int i) const {
        R v;
        load_real<L>(c + ((int64_t)i * 2 + part) * L, 1, v);
        return v;
    }
    XB_DEVICE R ld_part_cg(const double* c, int i, int p) const {
        double t[L];
#pragma unroll
        for (int l = 0; l < L; ++l) t[l] = __ldcg(c + ((int64_t)i * 2 + p) * L + l);
        R v;
        load_real<L>(t, 1, v);
        return v;
    }
    XB_DEVICE C ld_row(const double* c, int i) const {
        C z;
        load_real<L>(c + (int64_t)i * L2, 1, z.re);
        load_real<L>(c + (int64_t)i * L2 + L, 1, z.im);
        return z;
    }
    XB_DEVICE void st_part(double* c, int i, const R& v) const {
        store_real<L>(c + ((int64_t)i * 2 + part) * L, 1, v);
    }
};

// Local staging area for the cluster's warp partials (up to 8 CTAs x 4 warps
// x 2 halves x 4 limbs; two columns for the paired tree).
XB_DEVICE double* g2_stage() {
    __shared__ double s_stage[2 * 8 * 4 * 2 * 4];
    return s_stage;
}
// stage[(r*kG2Warps + w)*2L + part*L + l] = CTA r's slot[buf][w][part][l]
template <int L, class G2>
XB_DEVICE void g2_stage_partials(const G2& g, double* slot_local, int buf, int np, double* stage) {
    namespace cg = cooperative_groups;
    constexpr int W = 2 * L;  // doubles per warp partial
    for (int e = g.tid; e < np * W; e += kG2Threads) {
        const int r = e / (kG2Warps * W), rem = e % (kG2Warps * W);
        stage[e] = cg::this_cluster().map_shared_rank(slot_local, r)[buf * kG2Warps * W + rem];
    }
    __syncthreads();
}

// Cluster-wide fixed-order tree.  `acc` = this lane's in-lane partial (rows of
// its pair; `have` = the pair owns at least one row).  Levels: lane pairs of a
// warp (shuffle offsets 2, 4, 8, 16), then the cluster's 4*CS warp partials
// through DSMEM (each warp redoes the top levels, so every lane ends with the
// total of its own half; the other half is one shuffle away).
template <int L, int RPP>
XB_DEVICE real_t<L> g2_tree(const g2<L, RPP>& g, real_t<L> acc, double* slot_local, int buf) {
    namespace cg = cooperative_groups;
    using R = real_t<L>;
    const int pi = g.lane >> 1;
    // rolled loops: one copy of the add code, reused level after level (a
    // single warp running straight-line code is instruction-fetch bound)
#pragma unroll 1
    for (int s = 1; s < 16; s <<= 1) {
        R other = shfl_down_r(acc, 2 * s);
        if ((pi & (2 * s - 1)) == 0 && (g.gpair + s) * RPP < g.m) acc = addc(acc, other);
    }
    // slot[buf][warp][part] : L doubles
    double* my = slot_local + ((buf * kG2Warps + g.warp) * 2) * L;
    if (pi == 0) store_real<L>(my + g.part * L, 1, acc);
    cg::this_cluster().sync();
    const int np = kG2Warps * g.cs;          // warp partials in the cluster
    const int npp = np > 16 ? np / 16 : 1;   // partials per pair (1 or 2)
    const int rows_pp = 16 * RPP;            // rows covered by one warp partial
    // stage the cluster's partials in local shared memory, one DSMEM load per
    // thread (every warp reading every remote partial itself queues up
    // hundreds of DSMEM requests per CTA)
    double* stage = g2_stage();
    g2_stage_partials<L>(g, slot_local, buf, np, stage);
    R v = acc;
    int have = 0;
    R st0 = acc;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        if (u >= npp) break;
        const int k = pi * npp + u;
        if (k < np && k * rows_pp < g.m) {
            R w;
            load_real<L>(stage + (k * 2 + g.part) * L, 1, w);
            if (u == 0) {
                st0 = w;
                have = 1;
            } else {
                st0 = addc(st0, w);  // in-lane level (stride 1 partial)
            }
        }
    }
    v = st0;
#pragma unroll 1
    for (int s = 1; s < 16; s <<= 1) {
        R other = shfl_down_r(v, 2 * s);
        if ((pi & (2 * s - 1)) == 0 && (pi + s) * npp * rows_pp < g.m) v = addc(v, other);
    }
    (void)have;
    return shfl_idx_r(v, g.lane & 1);  // lane 0 holds re (or the real total), lane 1 im
}

// Two independent qd adds in lockstep as ONE call (add2_r4: both fast paths
// interleave): the bulk updates of two trailing columns share every level of
// their trees, at about the latency of one.
XB_CALL_IF rpair<r4> addc2(const r4 a1, const r4 b1, const r4 a2, const r4 b2) {
    return add2_r4(a1, b1, a2, b2);
}
XB_DEVICE rpair<r2> addc2(const r2& a1, const r2& b1, const r2& a2, const r2& b2) {
    return add2(a1, b1, a2, b2);
}
template <class R>
XB_DEVICE rpair<R> vadd(const rpair<R>& a, const rpair<R>& b) { return addc2(a.x, b.x, a.y, b.y); }
// the stored part of a reciprocal prefix (recip_t, xarith.cuh)
XB_DEVICE r2& rc_part(recip_t<r2>& rc) { return rc.x1; }
XB_DEVICE r4& rc_part(recip_t<r4>& rc) { return rc.x; }

// g2_tree for two columns at once (same pairing, same operands per column);
// slots: one per column, same double buffering.
template <int L, int RPP>
XB_DEVICE rpair<real_t<L>> g2_tree2(const g2<L, RPP>& g, rpair<real_t<L>> acc, double* slot_a,
                                    double* slot_b, int buf) {
    namespace cg = cooperative_groups;
    using R = real_t<L>;
    const int pi = g.lane >> 1;
#pragma unroll 1
    for (int s = 1; s < 16; s <<= 1) {
        const R o1 = shfl_down_r(acc.x, 2 * s), o2 = shfl_down_r(acc.y, 2 * s);
        if ((pi & (2 * s - 1)) == 0 && (g.gpair + s) * RPP < g.m) acc = addc2(acc.x, o1, acc.y, o2);
    }
    const int off = ((buf * kG2Warps + g.warp) * 2 + g.part) * L;
    if (pi == 0) {
        store_real<L>(slot_a + off, 1, acc.x);
        store_real<L>(slot_b + off, 1, acc.y);
    }
    cg::this_cluster().sync();
    const int np = kG2Warps * g.cs;
    const int npp = np > 16 ? np / 16 : 1;
    const int rows_pp = 16 * RPP;
    double* stage = g2_stage();
    double* stage_b = stage + 8 * kG2Warps * 2 * 4;
    {
        constexpr int W = 2 * L;
        for (int e = g.tid; e < np * W; e += kG2Threads) {
            const int r = e / (kG2Warps * W), rem = e % (kG2Warps * W);
            stage[e] = cg::this_cluster().map_shared_rank(slot_a, r)[buf * kG2Warps * W + rem];
            stage_b[e] = cg::this_cluster().map_shared_rank(slot_b, r)[buf * kG2Warps * W + rem];
        }
        __syncthreads();
    }
    rpair<R> v = acc;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        if (u >= npp) break;
        const int k = pi * npp + u;
        if (k < np && k * rows_pp < g.m) {
            R wa, wb;
            load_real<L>(stage + (k * 2 + g.part) * L, 1, wa);
            load_real<L>(stage_b + (k * 2 + g.part) * L, 1, wb);
            if (u == 0) {
                v.x = wa;
                v.y = wb;
            } else {
                v = addc2(v.x, wa, v.y, wb);
            }
        }
    }
#pragma unroll 1
    for (int s = 1; s < 16; s <<= 1) {
        const R o1 = shfl_down_r(v.x, 2 * s), o2 = shfl_down_r(v.y, 2 * s);
        if ((pi & (2 * s - 1)) == 0 && (pi + s) * npp * rows_pp < g.m) v = addc2(v.x, o1, v.y, o2);
    }
    return {shfl_idx_r(v.x, g.lane & 1), shfl_idx_r(v.y, g.lane & 1)};
}

template <int L, int RPP, bool LSQ>
__global__ void __launch_bounds__(kG2Threads, 2) mgs_grid2_kernel(GridParams p) {
    namespace cg = cooperative_groups;
    using R = real_t<L>;
    using C = cx<R>;
    constexpr int L2 = 2 * L;

    __shared__ double slot[2 * kG2Warps * 2 * L];
    __shared__ double slot2[2 * kG2Warps * 2 * L];  // second column of a paired update
    __shared__ int s_flag;

    g2<L, RPP> g;
    g.m = p.m;
    g.n = p.n;
    g.ncol = p.n + (LSQ ? 1 : 0);
    g.cs = p.cs;
    g.crank = (int)cg::this_cluster().block_rank();
    g.tid = threadIdx.x;
    g.lane = g.tid & 31;
    g.warp = g.tid >> 5;
    g.part = g.lane & 1;
    g.pair = g.warp * 16 + (g.lane >> 1);
    g.gpair = g.crank * kG2Pairs + g.pair;
    g.row0 = g.gpair * RPP;
    {
        int c = g.m - g.row0;
        g.cnt = c < 0 ? 0 : (c > RPP ? RPP : c);
    }
    g.ws = p.ws;
    const int m = g.m, n = g.n, ncol = g.ncol;
    const int cid = blockIdx.x / g.cs, G = gridDim.x / g.cs;
    int buf = 0;

    double* rdst = LSQ ? p.rws : p.r;
    double* ydst = LSQ ? p.rws + (int64_t)n * n * L2 : nullptr;
    auto record = [&](long long pos, int column, int code) {
        atomicMin(p.key, status_key(pos, column, code));
    };

    if (p.trace && blockIdx.x == 0 && g.tid == 0) p.trace[n * 8 + 7] = g2_timer();
    // ---- copy owned columns into the workspace (AoS image); QR: zero strict lower R
    for (int j = cid; j < ncol; j += G) {
        const double* src = (j < n) ? p.a + (int64_t)j * m * L2 : p.b;
        double* dst = g.col(j);
        for (int e = g.crank * kG2Threads + g.tid; e < m * L2; e += g.cs * kG2Threads) dst[e] = src[e];
        if (!LSQ && j < n && g.crank == 0)
            for (int e = j + 1 + g.tid; e < n; e += kG2Threads)
                for (int l = 0; l < L2; ++l) rdst[((int64_t)j * n + e) * L2 + l] = 0.0;
    }
    cg::this_cluster().sync();

    // ---- norm pre-pass (mgs.hpp:91-96 / :143): column_norm of every column --
    auto col_norm2 = [&](const double* c) -> R {
        R acc = lane_tree<(RPP >= 4 ? 3 : 2), R>(g.cnt, [&](int t) {
            C a = g.ld_row(c, g.row0 + t);
            return cdot_re(a, a);
        });
        R s = g2_tree<L, RPP>(g, acc, slot, buf);
        buf ^= 1;
        return s;
    };
    for (int j = cid; j < ncol; j += G) {
        R s = col_norm2(g.col(j));
        R nrm = rsqrt_ref(s);
        if (g.crank == 0 && g.tid == 0) {
            const bool bad = !vfinite(s) || !vfinite(nrm);
            if (bad) record(0, 0, XQR_OVERFLOW);
            store_real<L>(p.norms + (int64_t)j * L, 1, nrm);
            // the failure also travels in the norm (a NaN head): every CTA
            // derives the pre-pass verdict from data fixed before the
            // arrival barrier (p.key keeps changing after it)
            if (bad) p.norms[(int64_t)j * L] = __longlong_as_double(0x7ff8000000000000ll);
        }
    }
    // grid-wide arrival (all CTAs are co-resident: cooperative launch)
    __syncthreads();
    if (g.tid == 0) {
        __threadfence();
        g2_red_release(p.counters, 1);
        while (g2_ld_acquire(p.counters) < (int)gridDim.x) __nanosleep(64);
    }
    __syncthreads();
    R thr;
    bool pre_err = false;  // every thread reads every norm: uniform
    {
        R best = rmake<R>(0.0);
        for (int j = 0; j < ncol; ++j) {
            double t[L];
#pragma unroll
            for (int l = 0; l < L; ++l) t[l] = __ldcg(p.norms + (int64_t)j * L + l);
            R v;
            load_real<L>(t, 1, v);
            if (L > 1 && t[0] != t[0]) pre_err = true;  // (double is unchecked)
            if (lt(best, v)) best = v;
        }
        // breakdown_threshold (mgs.hpp:66-70)
        thr = mul(rmake<R>((double)m * real_of<L>::eps), best);
    }
    // pivot flags: every CTA of the owner cluster adds 1 once q_j is out, or
    // kFlagErr + 1 if normalising column j failed in it; published when the
    // low half reaches cs.  A cluster stops only at a failed pivot's flag, so
    // every round before it still completes everywhere and the first error
    // in program order is recorded (an overflow in a bulk update is only
    // recorded: the column's own normalisation fails later)
    constexpr int kFlagErr = 0x10000;
    if (p.trace && blockIdx.x == 0 && g.tid == 0) p.trace[n * 8 + 2] = g2_timer();  // pre-pass done

    // normalise column j (owner cluster) and publish it.  Returns false on error.
    auto normalize_publish = [&](int j) -> bool {
        double* c = g.col(j);
        R s = col_norm2(c);
        const bool tr = p.trace && g.tid == 0 && g.crank == 0;
        if (tr) p.trace[j * 8 + 4] = g2_timer();
        // the scalar chain (sqrt, breakdown test, reciprocal) runs in warp 0
        // only; the other warps wait and leave their issue slots to the CTA
        // that shares the SM
        __shared__ double s_rkk[L], s_rc[L];
        __shared__ int s_code;
        if (g.warp == XB_CHAIN_WARP) {
            R rkk0 = rsqrt_ref(s);
            if (tr) p.trace[j * 8 + 5] = g2_timer();
            int code0 = 0;
            if (!vfinite(s) || !vfinite(rkk0))
                code0 = XQR_OVERFLOW;
            else if (le(rkk0, thr))
                code0 = XQR_BREAKDOWN;
            recip_t<R> rc0;
            if (!code0) {
                int stc = 0;
                rc0 = recip(rkk0, stc);
                code0 = stc;
            }
            if (g.lane == 0) {
                store_real<L>(s_rkk, 1, rkk0);
                if (!code0) store_real<L>(s_rc, 1, rc_part(rc0));
                s_code = code0;
            }
        }
        __syncthreads();
        R rkk;
        load_real<L>(s_rkk, 1, rkk);
        const int code = s_code;
        recip_t<R> rc;
        if (!code) load_real<L>(s_rc, 1, rc_part(rc));
        if (tr) p.trace[j * 8 + 6] = g2_timer();
        // code is cluster-uniform (same tree, same r_kk in every CTA); an
        // overflow while dividing rows is local: it is recorded and stops the
        // factorisation at the next round start, never in mid-round
        bool ok = true;
        if (!code) {
            for (int t = 0; t < g.cnt; ++t) {
                R v = divide(g.ld_part(c, g.row0 + t), rkk, rc);
                if (!vfinite(v)) ok = false;
                g.st_part(c, g.row0 + t, v);
            }
        }
        ok = __syncthreads_and(ok);
        if (tr) p.trace[j * 8 + 7] = g2_timer();
        if (g.tid == 0) {
            if (code || !ok) {
                record(1 + (long long)j * (ncol + 1), code == XQR_BREAKDOWN ? j + 1 : 0,
                       code ? code : XQR_OVERFLOW);
            } else if (g.crank == 0) {
                C d{rkk, rmake<R>(0.0)};
                store_aos<L>(rdst + ((int64_t)j * n + j) * L2, d);
            }
            // no separate fence: the release (after the CTA barrier) already
            // orders every thread's column writes before the flag (a
            // __threadfence here cost 0.25 us per pivot)
            g2_red_release(p.flags + j, (code || !ok) ? kFlagErr + 1 : 1);
            if (p.trace && g.crank == 0) p.trace[j * 8 + 2] = g2_timer();
        }
        return code == 0;
    };

    bool abort = pre_err;
    if (!abort && cid == 0) abort = !normalize_publish(0);

    // ---- MGS rounds ----------------------------------------------------------------
    for (int k = 0; k < n && !abort; ++k) {
        const int j0 = k + 1 + ((cid - (k + 1)) % G + G) % G;
        if (j0 >= ncol) continue;
        // cluster-uniform decision: rank 0 acquires q_k (or its failure), the
        // cluster barrier hands the verdict to every CTA
        if (g.crank == 0 && g.tid == 0) {
            int v;
            // back off while waiting: dozens of clusters polling the L2 flat
            // out slow down everyone's loads, the critical path first
            while (((v = *(volatile int*)(p.flags + k)) & (kFlagErr - 1)) < g.cs) __nanosleep(64);
            __threadfence();  // acquire side (pairs with the publisher's red.release)
            s_flag = v < kFlagErr ? 1 : 0;
        }
        cg::this_cluster().sync();
        // one DSMEM read per CTA, then a CTA broadcast (every thread reading
        // rank 0's word at once costs microseconds)
        __shared__ int s_go;
        if (g.tid == 0) s_go = *cg::this_cluster().map_shared_rank(&s_flag, 0);
        __syncthreads();
        if (s_go == 0) {
            abort = true;
            break;
        }
        // q_k rows of this lane pair, both halves, in registers
        C q[RPP];
        const double* qk = g.col(k);
#pragma unroll
        for (int t = 0; t < RPP; ++t)
            if (t < g.cnt) {
                q[t].re = g.ld_part_cg(qk, g.row0 + t, 0);
                q[t].im = g.ld_part_cg(qk, g.row0 + t, 1);
            }
        if (p.trace && g.tid == 0 && g.crank == 0 && j0 == k + 1) p.trace[(k + 1) * 8 + 0] = g2_timer();
        const long long pos_k = 1 + (long long)k * (ncol + 1);
        for (int j = j0; j < ncol; j += G) {
            if (p.pair_bulk && j != k + 1 && j + G < ncol) {
                // two trailing columns off the critical path, in lockstep:
                // per column exactly the single-column operations below
                const int j2 = j + G;
                double* c1 = g.col(j);
                double* c2 = g.col(j2);
                rpair<R> acc = lane_tree<(RPP >= 4 ? 3 : 2), rpair<R>>(g.cnt, [&](int t) {
                    const C a1 = g.ld_row(c1, g.row0 + t), a2 = g.ld_row(c2, g.row0 + t);
                    const rpair<R> p1 = mul2(q[t].re, g.part ? a1.im : a1.re, neg(q[t].im), g.part ? a1.re : a1.im);
                    const rpair<R> p2 = mul2(q[t].re, g.part ? a2.im : a2.re, neg(q[t].im), g.part ? a2.re : a2.im);
                    return addc2(p1.x, g.part ? p1.y : neg(p1.y), p2.x, g.part ? p2.y : neg(p2.y));
                });
                const rpair<R> rh = g2_tree2<L, RPP>(g, acc, slot, slot2, buf);
                buf ^= 1;
                const R ro1 = shfl_xor_r(rh.x, 1), ro2 = shfl_xor_r(rh.y, 1);
                C r1, r2;
                r1.re = g.part ? ro1 : rh.x;
                r1.im = g.part ? rh.x : ro1;
                r2.re = g.part ? ro2 : rh.y;
                r2.im = g.part ? rh.y : ro2;
                bool ok1 = vfinite(r1.re) && vfinite(r1.im), ok2 = vfinite(r2.re) && vfinite(r2.im);
                for (int t = 0; t < g.cnt; ++t) {
                    const R y1 = g.part ? q[t].im : q[t].re, y2 = g.part ? q[t].re : q[t].im;
                    const rpair<R> pa = mul2(r1.re, y1, r1.im, y2);
                    const rpair<R> pb = mul2(r2.re, y1, r2.im, y2);
                    const rpair<R> tt = addc2(pa.x, g.part ? pa.y : neg(pa.y), pb.x, g.part ? pb.y : neg(pb.y));
                    const rpair<R> v = addc2(g.ld_part(c1, g.row0 + t), neg(tt.x), g.ld_part(c2, g.row0 + t),
                                             neg(tt.y));
                    if (!vfinite(v.x)) ok1 = false;
                    if (!vfinite(v.y)) ok2 = false;
                    g.st_part(c1, g.row0 + t, v.x);
                    g.st_part(c2, g.row0 + t, v.y);
                }
                ok1 = __syncthreads_and(ok1);
                ok2 = __syncthreads_and(ok2);
                if (g.tid < 2 && g.crank == 0) {
                    double* d1 = rdst + ((int64_t)j * n + k) * L2;
                    double* d2 = (j2 < n) ? rdst + ((int64_t)j2 * n + k) * L2 : ydst + (int64_t)k * L2;
                    store_real<L>(d1 + g.part * L, 1, rh.x);
                    store_real<L>(d2 + g.part * L, 1, rh.y);
                    if (!ok1 && g.tid == 0) record(pos_k + (j - k), 0, XQR_OVERFLOW);
                    if (!ok2 && g.tid == 0) record(pos_k + (j2 - k), 0, XQR_OVERFLOW);
                }
                j = j2;  // the loop's j += G moves past the pair
                continue;
            }
            double* c = g.col(j);
            // r_kj = q_k^H a_j (reduction.hpp:45-51): this lane's half of the
            // complex leaf cmul(conj(q), a) (complex.hpp:41-44), operands
            // selected so both halves run the same code
            R acc = lane_tree<(RPP >= 4 ? 3 : 2), R>(g.cnt, [&](int t) {
                C a = g.ld_row(c, g.row0 + t);
                const R y1 = g.part ? a.im : a.re, y2 = g.part ? a.re : a.im;
                rpair<R> pr = mul2(q[t].re, y1, neg(q[t].im), y2);
                return add(pr.x, g.part ? pr.y : neg(pr.y));
            });
            R rh = g2_tree<L, RPP>(g, acc, slot, buf);
            buf ^= 1;
            C r;
            R ro = shfl_xor_r(rh, 1);
            r.re = g.part ? ro : rh;
            r.im = g.part ? rh : ro;
            bool ok = vfinite(r.re) && vfinite(r.im);
            // a_i -= r * q_i (mgs.hpp:59): t = cmul(r, q_i), a - t
            for (int t = 0; t < g.cnt; ++t) {
                const R y1 = g.part ? q[t].im : q[t].re, y2 = g.part ? q[t].re : q[t].im;
                rpair<R> pr = mul2(r.re, y1, r.im, y2);
                R tt = add(pr.x, g.part ? pr.y : neg(pr.y));
                R v = sub(g.ld_part(c, g.row0 + t), tt);
                if (!vfinite(v)) ok = false;
                g.st_part(c, g.row0 + t, v);
            }
            ok = __syncthreads_and(ok);
            if (g.tid < 2 && g.crank == 0) {
                // lanes 0 / 1 hold re / im of r; write r_kj (or y_k)
                double* dst = (j < n) ? rdst + ((int64_t)j * n + k) * L2 : ydst + (int64_t)k * L2;
                store_real<L>(dst + g.part * L, 1, rh);
                if (!ok && g.tid == 0) record(pos_k + (j - k), 0, XQR_OVERFLOW);
            }
            if (p.trace && g.tid == 0 && g.crank == 0 && j == k + 1) p.trace[(k + 1) * 8 + 1] = g2_timer();
            if (j == k + 1 && j < n) {
                if (!normalize_publish(j)) {
                    abort = true;
                    break;
                }
            }
        }
        if (p.trace && g.tid == 0) atomicMax(p.trace + (k + 1) * 8 + 3, g2_timer());
    }

    // z = column_norm(b) by its owner (mgs.hpp:155)
    if (LSQ && !abort && (n % G) == cid) {
        R s = col_norm2(g.col(n));
        R z = rsqrt_ref(s);
        if (g.tid == 0 && g.crank == 0) {
            if (!vfinite(s) || !vfinite(z)) record(1 + (long long)n * (ncol + 1), 0, XQR_OVERFLOW);
            store_real<L>(p.z, 1, z);
        }
    }
    if (!LSQ) {
        // Q = the normalised owned columns (the workspace is the AoS image)
        // (each lane copies the halves it wrote itself: no cluster barrier needed)
        for (int j = cid; j < n; j += G) {
            const double* src = g.col(j);
            double* dst = p.q + (int64_t)j * m * L2;
            for (int t = 0; t < g.cnt; ++t) g.st_part(dst, g.row0 + t, g.ld_part(src, g.row0 + t));
        }
    }
    // no CTA may exit while a cluster peer can still read its shared memory
    cg::this_cluster().sync();
    // the status so far; a least-squares solve continues in
    // grid2_backsub_kernel (same stream) with more threads than a CTA here
    __syncthreads();
    if (g.tid == 0) {
        __threadfence();
        g2_red_release(p.counters + 1, 1);
    }
    if (blockIdx.x == 0 && g.tid == 0) {
        while (g2_ld_acquire(p.counters + 1) < (int)gridDim.x) __nanosleep(64);
        const unsigned long long key = __ldcg(p.key);
        if (p.trace) p.trace[n * 8 + 4] = g2_timer();
        xqr_status st;
        st.system = p.sys;
        st.code = key == kNoError ? 0 : (int)(key & 15);
        st.column = key == kNoError ? 0 : (int)((key >> 4) & 0xFFFFF);
        *p.st = st;
    }
}

// Back substitution of the single-system least-squares solve (mgs.hpp:157 ->
// :110-126): one CTA of kG2BsThreads threads, one lane pair per unknown for
// n <= 256 warp-specialised (flow_back_substitute): a finisher warp runs the
// chain, updater warps trail it; no CTA barrier per step.
#ifndef XB_G2BS_THREADS
#define XB_G2BS_THREADS 512
#endif
constexpr int kG2BsThreads = XB_G2BS_THREADS;
template <int L>
__host__ __device__ constexpr bool g2_backsub_prep_in_smem(int n) {
    // 227 KB less the static merge slots (XB_XSMEM) and the flags
    return sizeof(double) * (size_t)n * (2 * L + 3 * L + 1) <= 227 * 1024 - 64 * XB_XS_THREADS - 1024;
}
template <int L>
__host__ __device__ constexpr size_t g2_backsub_smem(int n) {
    return sizeof(double) * (size_t)n * (g2_backsub_prep_in_smem<L>(n) ? 2 * L + 3 * L + 1 : 2 * L);
}
template <int L>
__global__ void __launch_bounds__(kG2BsThreads, 1) grid2_backsub_kernel(GridParams p) {
    constexpr int L2 = 2 * L;
    extern __shared__ double xs[];
    __shared__ unsigned long long s_key;
    __shared__ int s_sync[2 + 32];
    const int n = p.n, ncol = n + 1;
    if (threadIdx.x == 0) s_key = *p.key;
    __syncthreads();
    if (s_key != kNoError) return;  // status already written by the factorisation
    if (p.trace && threadIdx.x == 0) p.trace[n * 8 + 5] = g2_timer();
    const double* ydst = p.rws + (int64_t)n * n * L2;
    // the Smith records in shared memory when they fit, else in the global
    // scratch after y (n > ~1300 quad-double unknowns)
    double* prep = g2_backsub_prep_in_smem<L>(n) ? xs + (size_t)n * L2 : p.rws + (int64_t)n * n * L2 + (int64_t)n * L2;
    bool bad = flow_back_substitute<L>(n, p.rws, ydst, xs, prep, s_sync, &s_key,
                                       2 + (long long)n * (ncol + 1), p.trace ? p.trace + 8 * (n + 1) : nullptr);
    if (!bad)
        for (int e = threadIdx.x; e < n * L2; e += blockDim.x) p.x[e] = xs[e];
    __syncthreads();
    if (p.trace && threadIdx.x == 0) p.trace[n * 8 + 6] = g2_timer();
    if (threadIdx.x == 0 && s_key != kNoError) {
        xqr_status st;
        st.system = p.sys;
        st.code = (int)(s_key & 15);
        st.column = (int)((s_key >> 4) & 0xFFFFF);
        *p.st = st;
    }
}

template <int L, int RPP, bool LSQ>
cudaError_t launch_grid2_t(const GridParams& p, int max_clusters, cudaStream_t s) {
    auto kern = mgs_grid2_kernel<L, RPP, LSQ>;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.blockDim = dim3(kG2Threads, 1, 1);
    // x of the back substitution lives here (CTA 0); the size also keeps the
    // kernel at ONE CTA per SM, so each warp has an SM sub-partition to itself
    cfg.dynamicSmemBytes = sizeof(double) * (size_t)p.n * 2 * L;
    {
        // CTAs per SM (kGrid2PerSM; XQR_GRID_PER_SM overrides, dev only)
        const char* e = std::getenv("XQR_GRID_PER_SM");
        const int per_sm = e ? std::max(1, std::atoi(e)) : kGrid2PerSM;
        size_t floor_b = per_sm == 1 ? 120 * 1024 : (per_sm == 2 ? 100 * 1024 : 60 * 1024);
        // the floor counts the kernel's static shared memory too
        cudaFuncAttributes fa;
        if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess) floor_b -= std::min(floor_b, fa.sharedSizeBytes);
        if (cfg.dynamicSmemBytes < floor_b) cfg.dynamicSmemBytes = floor_b;
    }
    {  // (static + dynamic may pass 48 KB even when the dynamic part does not)
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)cfg.dynamicSmemBytes);
        if (e != cudaSuccess) return e;
    }
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    // dev: XQR_NO_COOP=1 drops the cooperative attribute (same grid, all CTAs
    // still co-resident in practice) so a profiler that cannot replay
    // cooperative cluster launches can capture the kernel
    if (const char* e = std::getenv("XQR_NO_COOP"))
        if (e[0] == '1') cfg.numAttrs = 1;
    // as many clusters as fit co-resident (and no more than there are columns)
    int nclusters = 0;
    cfg.gridDim = dim3(p.cs, 1, 1);
    if (p.cs > 8) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, (void*)kern, &cfg);
    if (e != cudaSuccess) return e;
    const int ncol = p.n + (LSQ ? 1 : 0);
    if (nclusters > max_clusters) nclusters = max_clusters;
    if (nclusters > ncol) nclusters = ncol;
    if (nclusters < 1) return cudaErrorInvalidConfiguration;
    cfg.gridDim = dim3(nclusters * p.cs, 1, 1);
    return cudaLaunchKernelEx(&cfg, kern, p);
}

// The back substitution of a least-squares solve, launched after the grid
// kernel on the same stream.
template <int L>
cudaError_t launch_grid2_backsub(const GridParams& p, cudaStream_t s) {
    auto bs = grid2_backsub_kernel<L>;
    const size_t bsmem = g2_backsub_smem<L>(p.n);
    {  // (static + dynamic may pass 48 KB even when the dynamic part does not)
        cudaError_t e = cudaFuncSetAttribute(bs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem);
        if (e != cudaSuccess) return e;
    }
    bs<<<1, kG2BsThreads, bsmem, s>>>(p);
    return cudaGetLastError();
}

// RPP = 1 (m <= 256) and RPP = 2, 4 (m <= 1024) are instantiated in
// separate translation units (mgs_grid_L4.cu, mgs_grid_L4w.cu) so each can be
// compiled with the call-form mix it is fastest with (Makefile).
template <int L, int RPP>
cudaError_t launch_grid2_rpp(const GridParams& p, bool lsq, int max_clusters, cudaStream_t s) {
    return lsq ? launch_grid2_t<L, RPP, true>(p, max_clusters, s)
               : launch_grid2_t<L, RPP, false>(p, max_clusters, s);
}

}  // namespace xb
