// xmgs.cuh -- modified Gram-Schmidt QR / least squares, one CTA per system.
//
// Reference: mgs_qr (mgs.hpp:84-106), lsq_solve (mgs.hpp:131-158),
// back_substitute (mgs.hpp:110-126), with the reference's own decomposition
// (parallel.hpp:54-84: one round per pivot, one task per trailing column)
// mapped onto a CTA:
//   * a column task = one warp (lane owns consecutive rows, xcolumn.cuh);
//   * warps pull trailing columns from a shared-memory counter, so the pivot
//     normalisation (the longest task) never stalls a whole round;
//   * look-ahead: whichever warp draws column k+1 in round k normalises it as
//     soon as its projection is removed and publishes q_{k+1} in the other
//     shared-memory pivot slot -- round k+1 starts with its pivot ready;
//   * the right-hand side rides along as column n and is never normalised
//     (mgs.hpp:153); y and z stay on the device and feed the fused back
//     substitution (xbacksub.cuh).
// The pivot is normalised once (the reference's `designated` mode,
// parallel.hpp:55-59); the `redundant` mode gives identical bits
// (test_parallel.cpp:116-131), so one device path serves both.
#pragma once
#include "xbacksub.cuh"
#include "xcolumn.cuh"
#include "xpair.cuh"
#include "xqr_internal.h"

namespace xb {

// LV = depth of the in-lane tree stack: rows-per-lane <= 2^(LV-1).
template <int L, int LV>
struct mgs_warp {
    static constexpr int LIMBS = L;
    using R = real_t<L>;
    using C = cx<R>;
    using F = colfmt<L>;

    XB_DEVICE static int lane_rows(int lane, int m, int rpl) {
        int c = m - lane * rpl;
        return c < 0 ? 0 : (c > rpl ? rpl : c);
    }

    // Re(a^H a) over the fixed tree (mgs.hpp:38-42, reduction.hpp:45-51);
    // result broadcast to every lane.
    XB_DEVICE static R col_sq(const F& f, const double* col, int lane, int m) {
        const int cnt = lane_rows(lane, m, f.rpl);
        R acc = lane_tree<LV, R>(cnt, [&](int t) {
            C a = f.load(col, t, lane);
            return cdot_re(a, a);
        });
        acc = warp_tree(acc, lane, m, f.rpl);
        return shfl_idx_r(acc, 0);
    }

    // q^H a over the fixed tree; broadcast.
    XB_DEVICE static C dot(const F& f, const double* q, const double* col, int lane, int m) {
        const int cnt = lane_rows(lane, m, f.rpl);
        C acc = lane_tree<LV, C>(cnt, [&](int t) {
            return cmul(cconj(f.load(q, t, lane)), f.load(col, t, lane));
        });
        acc = warp_tree(acc, lane, m, f.rpl);
        return shfl_idx_c(acc, 0);
    }

    // remove_projection (mgs.hpp:57-61): r = q^H a; a_i -= r * q_i.
    // Returns false if any produced value is not finite.
    XB_DEVICE static bool remove_projection(const F& f, const double* q, double* col, int lane, int m,
                                         C& r) {
        r = dot(f, q, col, lane, m);
        bool ok = cfinite(r);
        const int cnt = lane_rows(lane, m, f.rpl);
#pragma unroll 1
        for (int t = 0; t < cnt; ++t) {
            C a = f.load(col, t, lane);
            a = csub(a, cmul(r, f.load(q, t, lane)));
            ok = ok && cfinite(a);
            f.store(col, t, lane, a);
        }
        return __all_sync(0xffffffffu, ok);
    }

    // normalize_column (mgs.hpp:46-53) into col and the shared pivot slot.
    // code: 0 ok, 1 breakdown, 2 overflow, 3 domain.
    XB_DEVICE static int normalize(const F& f, double* col, double* slot, const R& thr, int lane, int m,
                                R& rkk) {
        R s = col_sq(f, col, lane, m);
        rkk = rsqrt_ref(s);
        if (!vfinite(s) || !vfinite(rkk)) return 2;
        if (le(rkk, thr)) return 1;
        int st = 0;
        recip_t<R> rc = recip(rkk, st);
        if (st) return st;
        const int cnt = lane_rows(lane, m, f.rpl);
        bool ok = true;
#pragma unroll 1
        for (int t = 0; t < cnt; ++t) {
            C a = f.load(col, t, lane);
            C q = cdivide_real(a, rkk, rc);
            ok = ok && cfinite(q);
            f.store(col, t, lane, q);
            f.store(slot, t, lane, q);
        }
        return __all_sync(0xffffffffu, ok) ? 0 : 2;
    }
};

// quad-double batches: the warp-specialised back substitution of the
// single-system path (xbacksub.cuh) instead of the barrier-per-step sweep
// (4096 x cqd 128x128: 870 -> 863 ms, same bits)
#ifndef XB_CTA_FLOW_BS
#define XB_CTA_FLOW_BS 1
#endif

// W = the column primitives: mgs_warp<L, LV> (a lane per row group,
// xcolumn.cuh) or mgs_pair<L> (a lane pair per row group, xpair.cuh).
template <class W, int NW, bool LSQ, int MINB = 1>
__global__ void __launch_bounds__(NW * 32, MINB) mgs_cta_kernel(SolveParams p, int rpl) {
    constexpr int L = W::LIMBS;
    using R = real_t<L>;
    using C = cx<R>;
    constexpr int L2 = 2 * L;
    const typename W::F f(rpl);

    extern __shared__ double smem[];  // two pivot slots of f.COL doubles
    __shared__ unsigned long long s_key;
    __shared__ int s_ctr[2];
    __shared__ R s_best[NW];
    __shared__ double s_hmax[NW];
    __shared__ R s_thr;
    __shared__ R s_z;

    const int64_t sys = blockIdx.x;
    const int m = p.m, n = p.n;
    const int ncol = n + (LSQ ? 1 : 0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nt = blockDim.x;
    double* ws = p.ws + sys * p.ws_stride;
    double* rws = LSQ ? p.rws + sys * p.rws_stride : nullptr;
    // R destination: QR -> the caller's AoS r; LS -> device scratch
    double* rdst = LSQ ? rws : p.r + sys * (int64_t)n * n * L2;
    double* ydst = LSQ ? rws + (int64_t)n * n * L2 : nullptr;

    // ---- pack AoS -> lane-interleaved planar -------------------------------
    {
        const double* A = p.a + sys * (int64_t)m * n * L2;
        const int64_t tot = (int64_t)m * n * L2;
        for (int64_t e = threadIdx.x; e < tot; e += nt) {
            const int plane = (int)(e % L2);
            const int64_t ij = e / L2;
            const int i = (int)(ij % m), j = (int)(ij / m);
            ws[(int64_t)j * f.COL + plane * f.LD + f.row_off(i)] = A[e];
        }
        if (LSQ) {
            const double* B = p.b + sys * (int64_t)m * L2;
            for (int e = threadIdx.x; e < m * L2; e += nt) {
                const int plane = e % L2, i = e / L2;
                ws[(int64_t)n * f.COL + plane * f.LD + f.row_off(i)] = B[e];
            }
        } else {
            // strictly lower triangle of R is +0 (mgs.hpp:87 col_matrix init)
            for (int64_t e = threadIdx.x; e < (int64_t)n * n; e += nt) {
                const int i = (int)(e % n), j = (int)(e / n);
                if (i > j)
                    for (int l = 0; l < L2; ++l) rdst[e * L2 + l] = 0.0;
            }
        }
        if (threadIdx.x == 0) {
            s_key = kNoError;
            s_ctr[0] = 0;
            s_ctr[1] = 0;
        }
    }
    __syncthreads();

    // ---- norm pre-pass and breakdown threshold (mgs.hpp:91-96, :143) --------
    // max_column_norm (mgs.hpp:72-80) = max_j sqrt(s_j), s_j = Re(a_j^H a_j).
    // The square roots are taken only where they can decide the maximum:
    // for the columns whose s_j is within a relative 2^-40 of the largest
    // (compared on the head limbs) -- sqrt is monotone up to its rounding
    // (double: exact; dd / qd: ~2^-104 / ~2^-208 relative, mgs.hpp / the
    // reference's sqrt), so a column further down can never hold the
    // largest norm, and the maximum of the rest is the reference's value
    // bit for bit -- plus the extreme magnitudes, whose square roots could
    // overflow on their own (the reference raises overflow_error there).
    bool err = false;
    {
        double* sb = smem;  // s_j (L doubles each) in the pivot slots, free until pivot 0
        double hmax = 0.0;
        for (int j = warp; j < ncol; j += NW) {
            const R s = W::col_sq(f, ws + (int64_t)j * f.COL, lane, m);
            if (!vfinite(s)) err = true;
            if (lane == 0) store_real<L>(sb + (int64_t)j * L, 1, s);
            hmax = fmax(hmax, s.c0);
        }
        if (lane == 0) {
            s_hmax[warp] = hmax;
            if (err) atomicMin(&s_key, status_key(0, 0, XQR_OVERFLOW));
        }
        if (__syncthreads_or(err)) goto finish;
        for (int w = 0; w < NW; ++w) hmax = fmax(hmax, s_hmax[w]);
        const double near = hmax * (1.0 - 0x1p-40);
        R best = rmake<R>(0.0);
        for (int j = warp; j < ncol; j += NW) {
            R s;
            load_real<L>(sb + (int64_t)j * L, 1, s);
            const double h = s.c0;
            if (h >= near || h > 0x1p1000 || (h != 0.0 && h < 0x1p-1000)) {
                const R nrm = rsqrt_ref(s);
                if (!vfinite(nrm)) err = true;
                if (lt(best, nrm)) best = nrm;
            }
        }
        if (lane == 0) {
            s_best[warp] = best;
            if (err) atomicMin(&s_key, status_key(0, 0, XQR_OVERFLOW));
        }
    }
    if (__syncthreads_or(err)) goto finish;
    if (threadIdx.x == 0) {
        R best = s_best[0];
        for (int w = 1; w < NW; ++w)
            if (lt(best, s_best[w])) best = s_best[w];
        // breakdown_threshold (mgs.hpp:66-70): R(rows * eps) * max_norm
        s_thr = mul(rmake<R>((double)m * real_of<L>::eps), best);
    }
    __syncthreads();

    {
        const R thr = s_thr;
        // pivot 0
        if (warp == 0) {
            R rkk;
            int code = W::normalize(f, ws, smem, thr, lane, m, rkk);
            if (code) {
                if (lane == 0) atomicMin(&s_key, status_key(1, 1, code));
                err = true;
            } else if (lane == 0) {
                store_aos<L>(rdst, C{rkk, rmake<R>(0.0)});
            }
        }
        if (__syncthreads_or(err)) goto finish;

        // ---- MGS rounds -------------------------------------------------------
        for (int k = 0; k < n; ++k) {
            if (threadIdx.x == 0) s_ctr[(k + 1) & 1] = 0;
            const double* qk = smem + (k & 1) * f.COL;
            const long long pos_k = 1 + (long long)k * (ncol + 1);
            for (;;) {
                int t = 0;
                if (lane == 0) t = atomicAdd(&s_ctr[k & 1], 1);
                t = __shfl_sync(0xffffffffu, t, 0);
                const int j = k + 1 + t;
                if (j >= ncol) break;
                double* col = ws + (int64_t)j * f.COL;
                C r;
                bool ok = W::remove_projection(f, qk, col, lane, m, r);
                if (!ok) {
                    if (lane == 0) atomicMin(&s_key, status_key(pos_k + (j - k), 0, XQR_OVERFLOW));
                    err = true;
                }
                if (lane == 0) {
                    if (j < n)
                        store_aos<L>(rdst + ((int64_t)j * n + k) * L2, r);
                    else
                        store_aos<L>(ydst + (int64_t)k * L2, r);
                }
                if (ok && j == k + 1 && j < n) {
                    R rkk;
                    int code = W::normalize(f, col, smem + (j & 1) * f.COL, thr, lane, m, rkk);
                    if (code) {
                        if (lane == 0)
                            atomicMin(&s_key,
                                      status_key(1 + (long long)j * (ncol + 1), j + 1, code));
                        err = true;
                    } else if (lane == 0) {
                        store_aos<L>(rdst + ((int64_t)j * n + j) * L2, C{rkk, rmake<R>(0.0)});
                    }
                }
            }
            if (__syncthreads_or(err)) goto finish;
        }

        if (LSQ) {
            // z = column_norm(b) (mgs.hpp:155)
            if (warp == 0) {
                R s = W::col_sq(f, ws + (int64_t)n * f.COL, lane, m);
                R z = rsqrt_ref(s);
                if (!vfinite(s) || !vfinite(z)) {
                    if (lane == 0)
                        atomicMin(&s_key,
                                  status_key(1 + (long long)n * (ncol + 1), 0, XQR_OVERFLOW));
                    err = true;
                }
                if (lane == 0) s_z = z;
            }
            if (__syncthreads_or(err)) goto finish;
            // back substitution (mgs.hpp:157 -> :110-126); x lives in the pivot
            // slots' shared memory (2*COL >= 2*2L*m >= 2L*n doubles)
            double* xs = smem;
            double* prep = rws + (int64_t)n * n * L2 + (int64_t)n * L2;
#if XB_CTA_FLOW_BS
            // quad-double: the warp-specialised sweep (finisher + updaters,
            // no CTA barrier per step), as for one large system
            if constexpr (L == 4) {
                __shared__ int s_sync[2 + NW];
                if (flow_back_substitute<L>(n, rws, ydst, xs, prep, s_sync, &s_key, 2 + (long long)n * (ncol + 1)))
                    goto finish;
            } else
#endif
            if (cta_back_substitute<L>(n, rws, ydst, xs, prep, &s_key,
                                       2 + (long long)n * (ncol + 1)))
                goto finish;
            double* X = p.x + sys * (int64_t)n * L2;
            for (int e = threadIdx.x; e < n * L2; e += nt) X[e] = xs[e];
            if (threadIdx.x == 0) store_real<L>(p.z + sys * L, 1, s_z);
        } else {
            // Q = the normalised columns (mgs.hpp:105): planar -> AoS
            double* Q = p.q + sys * (int64_t)m * n * L2;
            const int64_t tot = (int64_t)m * n * L2;
            for (int64_t e = threadIdx.x; e < tot; e += nt) {
                const int plane = (int)(e % L2);
                const int64_t ij = e / L2;
                const int i = (int)(ij % m), j = (int)(ij / m);
                Q[e] = ws[(int64_t)j * f.COL + plane * f.LD + f.row_off(i)];
            }
        }
    }

finish:
    if (threadIdx.x == 0) {
        unsigned long long key = s_key;
        xqr_status st;
        st.system = sys;
        if (key == kNoError) {
            st.code = 0;
            st.column = 0;
        } else {
            st.code = (int)(key & 15);
            st.column = (int)((key >> 4) & 0xFFFFF);
        }
        p.st[sys] = st;
    }
}

template <int L>
__global__ void __launch_bounds__(256) back_substitute_kernel(BackSubParams p) {
    extern __shared__ double smem[];
    __shared__ unsigned long long s_key;
    constexpr int L2 = 2 * L;
    const int64_t sys = blockIdx.x;
    const int n = p.n;
    if (threadIdx.x == 0) s_key = kNoError;
    __syncthreads();
    bool bad = cta_back_substitute<L>(n, p.r + sys * (int64_t)n * n * L2, p.y + sys * (int64_t)n * L2,
                                      smem, p.prep + sys * (int64_t)n * (3 * L + 1), &s_key, 0);
    if (!bad) {
        double* X = p.x + sys * (int64_t)n * L2;
        for (int e = threadIdx.x; e < n * L2; e += blockDim.x) X[e] = smem[e];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long key = s_key;
        xqr_status st;
        st.system = sys;
        st.code = key == kNoError ? 0 : (int)(key & 15);
        st.column = 0;
        p.st[sys] = st;
    }
}

}  // namespace xb
