// xgrid1.cuh -- single-system MGS QR / least squares over the whole GPU,
// double / double-double variant (cheap operations: a whole CTA per column,
// one thread per row, as many columns in flight as there are SMs).  The
// quad-double variant is xgrid2.cuh.
//
// One large system (the latency configs: cdd/cqd 256x256, cqd 512x256) is
// spread over a persistent cooperative grid, one 256-thread CTA per SM:
//   * column j (of [A b]) is owned by CTA j % G for the whole factorisation
//     (the reference's one-task-per-trailing-column round, parallel.hpp:60-67,
//     with the tasks pinned to SMs);
//   * a column task uses the whole CTA: thread t owns `rpt` consecutive rows,
//     so the fixed tree (reduction.hpp:34-40) is in-thread levels, then warp
//     shuffles, then the 8 warp partials reduced by warp 0 -- the same
//     pairing order as the sequential tree_reduce;
//   * the pivot q_k is published by its owner through global memory (it *is*
//     the finished column k) with a release flag; consumers acquire the flag
//     and stage q_k in shared memory.  There is no grid barrier per pivot;
//   * look-ahead: the owner of column k+1 updates it first in round k,
//     normalises it at once and publishes q_{k+1} while every other CTA is
//     still applying q_k to its trailing columns;
//   * the right-hand side is column n (never normalised); its owner computes
//     z, and after one grid barrier CTA 0 runs the fused back substitution.
// A pivot breakdown publishes an abort flag so no CTA waits forever; errors
// keep the reference's first-in-program-order semantics (status_key).
#pragma once
#include <cooperative_groups.h>
#include <cuda_pipeline.h>

#include "xbacksub.cuh"
#include "xcolumn.cuh"
#include "xqr_internal.h"

namespace xb {

constexpr int kGridThreads = 256;
constexpr int kGridWarps = kGridThreads / 32;


// Column layout for a CTA-wide task: plane stride LD = 256*rpt; row
// i*256 + t belongs to thread t's i-th consecutive row (coalesced).
template <int L>
struct gridfmt {
    int rpt, LD, COL;
    XB_DEVICE explicit gridfmt(int r) : rpt(r), LD(kGridThreads * r), COL(2 * L * kGridThreads * r) {}
    XB_DEVICE static int off(int i, int t) { return i * kGridThreads + t; }
    XB_DEVICE int row_off(int row) const { return (row % rpt) * kGridThreads + row / rpt; }
    XB_DEVICE cx<real_t<L>> load(const double* col, int i, int t) const {
        cx<real_t<L>> z;
        load_real<L>(col + off(i, t), LD, z.re);
        load_real<L>(col + L * LD + off(i, t), LD, z.im);
        return z;
    }
    XB_DEVICE cx<real_t<L>> load_cg(const double* col, int i, int t) const {
        // L2-coherent read of a column another CTA published
        cx<real_t<L>> z;
        const double* p = col + off(i, t);
        double v[2 * L];
#pragma unroll
        for (int l = 0; l < 2 * L; ++l) v[l] = __ldcg(p + l * LD);
        load_real<L>(v, 1, z.re);
        load_real<L>(v + L, 1, z.im);
        return z;
    }
    XB_DEVICE void store(double* col, int i, int t, const cx<real_t<L>>& z) const {
        store_real<L>(col + off(i, t), LD, z.re);
        store_real<L>(col + L * LD + off(i, t), LD, z.im);
    }
};

// CTA-wide tree over m rows: in-thread stack, warp shuffles, then the warp
// partials (strides 32*rpt, 64*rpt, 128*rpt) by warp 0.  Every thread gets
// the total.  `red` is a shared scratch of kGridWarps+1 values.
template <int LV, class V, class LeafFn>
XB_DEVICE V cta_tree(int m, int rpt, V* red, LeafFn leaf) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int cnt = m - tid * rpt;
    cnt = cnt < 0 ? 0 : (cnt > rpt ? rpt : cnt);
    V acc = lane_tree<LV, V>(cnt, leaf);
    // lanes: stride rpt*o <-> shuffle offset o; rows of lane (warp*32+lane)
    const int base = warp * 32;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        V other = vshfl_down(acc, o);
        if (((lane & (2 * o - 1)) == 0) && ((base + lane + o) * rpt < m)) acc = vadd(acc, other);
    }
    if (lane == 0 && base * rpt < m) red[warp] = acc;
    __syncthreads();
    if (warp == 0) {
        V w = acc;
        if (lane < kGridWarps && lane * 32 * rpt < m) w = red[lane];
#pragma unroll
        for (int o = 1; o < kGridWarps; o <<= 1) {
            V other = vshfl_down(w, o);
            if (((lane & (2 * o - 1)) == 0) && ((lane + o) * 32 * rpt < m)) w = vadd(w, other);
        }
        if (lane == 0) red[kGridWarps] = w;
    }
    __syncthreads();
    return red[kGridWarps];
}

XB_DEVICE unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
XB_DEVICE int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
XB_DEVICE void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Two columns' values in one tree pass (the chain mode's bulk CTAs update
// their columns in pairs: both reductions share every level's latency).
template <class C>
struct cpair {
    C x, y;
};
template <class C>
XB_DEVICE cpair<C> vadd(const cpair<C>& a, const cpair<C>& b) {
    return {vadd(a.x, b.x), vadd(a.y, b.y)};
}
template <class C>
XB_DEVICE cpair<C> vshfl_down(const cpair<C>& v, int o) {
    return {vshfl_down(v.x, o), vshfl_down(v.y, o)};
}

template <int L, int LV, bool LSQ>
__global__ void __launch_bounds__(kGridThreads, 1) mgs_grid_kernel(GridParams p) {
    namespace cg = cooperative_groups;
    using R = real_t<L>;
    using C = cx<R>;
    constexpr int L2 = 2 * L;
    const gridfmt<L> f(p.rpt);
    const int m = p.m, n = p.n;
    const int ncol = n + (LSQ ? 1 : 0);
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;

    extern __shared__ double smem[];  // q_k staging: f.COL doubles
    __shared__ C red_c[kGridWarps + 1];
    __shared__ cpair<C> red_p[kGridWarps + 1];
    __shared__ R red_r[kGridWarps + 1];
    __shared__ R s_thr;
    __shared__ int s_flag;

    double* rdst = LSQ ? p.rws : p.r;
    double* ydst = LSQ ? p.rws + (int64_t)n * n * L2 : nullptr;
    // dev trace, row n: 7 start, 4 factorised, 5/6 back substitution span
    if (p.trace && c == 0 && tid == 0) p.trace[n * 8 + 7] = gtimer();
    auto colp = [&](int j) { return p.ws + (int64_t)j * f.COL; };
    // Column ownership.  Cyclic mode: column j -> CTA j mod G, whose owner of
    // column k+1 updates it first in round k and normalises it.  Chain mode
    // (p.chain, G >= 3): CTA 0 owns no column but runs EVERY pivot -- the
    // last projection of column k+1 with q_k still in its shared memory, and
    // the normalisation -- alone on its SM, while CTAs 1.. own the columns
    // (j -> 1 + j mod (G-1)) and apply every earlier projection, reporting
    // each through p.cflags.  The chain then never waits for a pivot's
    // hand-off between CTAs.
    const bool chain = p.chain != 0 && G >= 3;
    const int S = chain ? G - 1 : G;         // ownership stride
    const int own0 = chain ? c - 1 : c;      // first owned column (< 0: none)
    const bool bulk = own0 >= 0;

    auto col_sq = [&](const double* col) {
        return cta_tree<LV, R>(m, f.rpt, red_r, [&](int i) {
            C a = f.load(col, i, tid);
            return cdot_re(a, a);
        });
    };
    auto record = [&](long long pos, int column, int code) {
        atomicMin(p.key, status_key(pos, column, code));
    };

    // ---- pack owned columns AoS -> planar; QR: zero the strict lower R -----
    for (int j = bulk ? own0 : ncol; j < ncol; j += S) {
        const double* src = (j < n) ? p.a + (int64_t)j * m * L2 : p.b;
        double* dst = colp(j);
        for (int e = tid; e < m * L2; e += kGridThreads) {
            const int plane = e % L2, i = e / L2;
            dst[plane * f.LD + f.row_off(i)] = src[e];
        }
        if (!LSQ && j < n)
            for (int e = j + 1 + tid; e < n; e += kGridThreads)
                for (int l = 0; l < L2; ++l) rdst[((int64_t)j * n + e) * L2 + l] = 0.0;
    }
    __syncthreads();

    // ---- norm pre-pass (mgs.hpp:91-96 / :143) ----------------------------------
    for (int j = bulk ? own0 : ncol; j < ncol; j += S) {
        R s = col_sq(colp(j));
        R nrm = rsqrt_ref(s);
        const bool bad = !vfinite(s) || !vfinite(nrm);
        if (tid == 0) {
            if (bad) record(0, 0, XQR_OVERFLOW);
            store_real<L>(p.norms + (int64_t)j * L, 1, nrm);
            // the failure also travels in the norm itself (a NaN head), so
            // every CTA derives the same pre-pass verdict from data fixed
            // before the grid barrier (p.key keeps changing after it)
            if (bad) p.norms[(int64_t)j * L] = __longlong_as_double(0x7ff8000000000000ll);
        }
    }
    cg::this_grid().sync();
    // every CTA computes the same max (order-independent), threshold and
    // pre-pass verdict
    bool pre_bad = false;
    {
        R best = rmake<R>(0.0);
        for (int j = tid; j < ncol; j += kGridThreads) {
            R v;
            const double* q = p.norms + (int64_t)j * L;
            double t[L];
#pragma unroll
            for (int l = 0; l < L; ++l) t[l] = __ldcg(q + l);
            load_real<L>(t, 1, v);
            if (L > 1 && t[0] != t[0]) pre_bad = true;  // (double is unchecked)
            if (lt(best, v)) best = v;
        }
        // CTA max (exact: the max is order-independent)
        const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            R other = shfl_down_r(best, o);
            if (lt(best, other)) best = other;
        }
        if (lane == 0) red_r[warp] = best;
        __syncthreads();
        if (tid == 0) {
            R b = red_r[0];
            for (int w = 1; w < kGridWarps; ++w)
                if (lt(b, red_r[w])) b = red_r[w];
            s_thr = mul(rmake<R>((double)m * real_of<L>::eps), b);
        }
        __syncthreads();
    }
    const R thr = s_thr;
    const bool pre_err = __syncthreads_or(pre_bad) != 0;  // grid-uniform: read from the norms

    // Chain mode: the next pivot column's own rows are copied into the spare
    // buffer with cp.async while the current pivot runs its scalar chain --
    // by each thread for its own rows, as soon as it sees the column's
    // earlier projections done (one acquire poll; if not yet, it loads them
    // itself when the pivot starts).  No other thread reads those rows.
    double* sc = smem + f.COL;            // the current pivot column
    double* sn = smem + 2 * (size_t)f.COL;  // the next one, in flight
    bool pref = false;
    auto chain_prefetch = [&](int jn) {
        pref = false;
        if (jn >= n || ld_acquire(p.cflags + jn) < jn - 1) return;
        const double* src = colp(jn);
        for (int i = 0; i < f.rpt; ++i)
            if (tid * f.rpt + i < m)
                for (int l = 0; l < 2 * L; ++l) {
                    const int o = f.off(i, tid) + l * f.LD;
                    __pipeline_memcpy_async(sn + o, src + o, sizeof(double));
                }
        __pipeline_commit();
        pref = true;
    };

    // normalise column j (owner) and publish it; returns false on error
    auto normalize_publish = [&](int j, double* col) -> bool {
        // chain mode: col is the chain's shared-memory copy; q_j also goes to
        // the staging area (the next pivot's q) and to the published column
        const bool copy_out = chain && col != colp(j);
        double* pcol = colp(j);
        const bool tr = p.trace && tid == 0;
        R s = col_sq(col);
        if (tr) p.trace[j * 8 + 4] = gtimer();
        R rkk = rsqrt_ref(s);
        if (tr) p.trace[j * 8 + 5] = gtimer();
        int code = 0;
        if (!vfinite(s) || !vfinite(rkk)) code = XQR_OVERFLOW;
        else if (le(rkk, thr)) code = XQR_BREAKDOWN;
        recip_t<R> rc;
        if (!code) {
            int stc = 0;
            rc = recip(rkk, stc);
            code = stc;
        }
        if (tr) p.trace[j * 8 + 6] = gtimer();
        // chain: the next pivot column, in flight during the divisions and
        // the publish (tried here rather than after the norm tree: the bulk
        // owner has had longer; measured 61 % ready at this point)
        if (copy_out) chain_prefetch(j + 1);
        bool ok = (code == 0);
        if (ok) {
            for (int i = 0; i < f.rpt; ++i) {
                if (tid * f.rpt + i < m) {
                    C a = f.load(col, i, tid);
                    C qv = cdivide_real(a, rkk, rc);
                    if (!cfinite(qv)) ok = false;
                    f.store(col, i, tid, qv);
                    if (copy_out) {
                        f.store(pcol, i, tid, qv);
                        f.store(smem, i, tid, qv);
                    }
                }
            }
        }
        ok = __syncthreads_and(ok);
        if (tr) p.trace[j * 8 + 7] = gtimer();
        if (tid == 0) {
            if (!ok) {
                record(1 + (long long)j * (ncol + 1), code == XQR_BREAKDOWN ? j + 1 : 0,
                       code ? code : XQR_OVERFLOW);
            } else {
                store_aos<L>(rdst + ((int64_t)j * n + j) * L2, C{rkk, rmake<R>(0.0)});
            }
            // no separate fence: the release (after the CTA barrier) already
            // orders every thread's column writes before the flag (a
            // __threadfence here cost 0.25 us per pivot)
            st_release(p.flags + j, ok ? 1 : 2);
            if (p.trace) p.trace[j * 8 + 2] = gtimer();
        }
        return ok;
    };

    // remove_projection(q_k, a_j) (mgs.hpp:57-61) with q_k staged in smem;
    // returns "all finite" (CTA-uniform)
    auto update_col = [&](int j, int k, double* col) -> bool {
        C r = cta_tree<LV, C>(m, f.rpt, red_c, [&](int i) {
            return cmul(cconj(f.load(smem, i, tid)), f.load(col, i, tid));
        });
        // dev trace: the critical update's dot product done (second stamp block)
        if (p.trace && tid == 0 && j == k + 1) p.trace[8 * (n + 1) + 8 * (k + 1)] = gtimer();
        bool ok = cfinite(r);
        for (int i = 0; i < f.rpt; ++i) {
            if (tid * f.rpt + i < m) {
                C a = f.load(col, i, tid);
                a = csub(a, cmul(r, f.load(smem, i, tid)));
                if (!cfinite(a)) ok = false;
                f.store(col, i, tid, a);
            }
        }
        ok = __syncthreads_and(ok);
        if (tid == 0) {
            if (!ok) record(1 + (long long)k * (ncol + 1) + (j - k), 0, XQR_OVERFLOW);
            if (j < n)
                store_aos<L>(rdst + ((int64_t)j * n + k) * L2, r);
            else
                store_aos<L>(ydst + (int64_t)k * L2, r);
        }
        return ok;
    };

    // two columns at once, per column exactly update_col's operations
    auto update_pair = [&](int j1, int j2, int k) {
        double* c1 = colp(j1);
        double* c2 = colp(j2);
        const cpair<C> rr = cta_tree<LV, cpair<C>>(m, f.rpt, red_p, [&](int i) {
            const C qc = cconj(f.load(smem, i, tid));
            return cpair<C>{cmul(qc, f.load(c1, i, tid)), cmul(qc, f.load(c2, i, tid))};
        });
        bool ok1 = cfinite(rr.x), ok2 = cfinite(rr.y);
        for (int i = 0; i < f.rpt; ++i) {
            if (tid * f.rpt + i < m) {
                const C qi = f.load(smem, i, tid);
                C a1 = f.load(c1, i, tid), a2 = f.load(c2, i, tid);
                a1 = csub(a1, cmul(rr.x, qi));
                a2 = csub(a2, cmul(rr.y, qi));
                if (!cfinite(a1)) ok1 = false;
                if (!cfinite(a2)) ok2 = false;
                f.store(c1, i, tid, a1);
                f.store(c2, i, tid, a2);
            }
        }
        ok1 = __syncthreads_and(ok1);
        ok2 = __syncthreads_and(ok2);
        if (tid == 0) {
            const long long pos_k = 1 + (long long)k * (ncol + 1);
            if (!ok1) record(pos_k + (j1 - k), 0, XQR_OVERFLOW);
            if (!ok2) record(pos_k + (j2 - k), 0, XQR_OVERFLOW);
            store_aos<L>(rdst + ((int64_t)j1 * n + k) * L2, rr.x);
            if (j2 < n)
                store_aos<L>(rdst + ((int64_t)j2 * n + k) * L2, rr.y);
            else
                store_aos<L>(ydst + (int64_t)k * L2, rr.y);
        }
    };

    bool abort = pre_err;
    auto chain_load = [&](int j) {  // own rows of column j (published by its owner) -> sc
        for (int i = 0; i < f.rpt; ++i)
            if (tid * f.rpt + i < m) f.store(sc, i, tid, f.load_cg(colp(j), i, tid));
    };
    if (!abort && c == 0) {
        if (chain) chain_load(0);
        abort = !normalize_publish(0, chain ? sc : colp(0));
    }
    if (pre_err && c == 0 && tid == 0) st_release(p.flags, 2);

    if (chain && c == 0) {
        // ---- the pivot chain: q_{j-1} staged in smem by this CTA's own
        // normalisation; column j's earlier projections from its owner
        for (int j = 1; j < n && !abort; ++j) {
            // column j: prefetched into sn during the last pivot, or loaded now
            if (pref) {
                __pipeline_wait_prior(0);
                double* t = sc;
                sc = sn;
                sn = t;
            } else {
                while (ld_acquire(p.cflags + j) < j - 1) __nanosleep(32);
                chain_load(j);
            }
            if (p.trace && tid == 0) p.trace[j * 8 + 0] = gtimer();
            const bool ok = update_col(j, j - 1, sc);
            if (p.trace && tid == 0) p.trace[j * 8 + 1] = gtimer();
            if (!ok) {
                if (tid == 0) st_release(p.flags + j, 2);
                abort = true;
                break;
            }
            if (!normalize_publish(j, sc)) {
                abort = true;
                break;
            }
        }
        __pipeline_wait_prior(0);  // nothing left in flight
    }

    // ---- MGS rounds ----------------------------------------------------------------
    for (int k = 0; k < n && !abort && bulk; ++k) {
        // first owned column > k (chain mode: the pivot column k+1 is the chain's)
        int j0 = k + 1 + ((own0 - (k + 1)) % S + S) % S;
        if (chain && j0 == k + 1 && j0 < n) j0 += S;
        if (j0 >= ncol) continue;
        // acquire q_k
        if (tid == 0) {
            int v;
            while ((v = ld_acquire(p.flags + k)) == 0) __nanosleep(32);
            s_flag = v;
        }
        __syncthreads();
        if (s_flag != 1) {
            abort = true;
            break;
        }
        {
            const double* qk = colp(k);
            for (int e = tid; e < f.COL; e += kGridThreads) smem[e] = __ldcg(qk + e);
        }
        __syncthreads();
        if (p.trace && tid == 0 && j0 == k + 1) p.trace[(k + 1) * 8 + 0] = gtimer();
        for (int j = j0; j < ncol; j += S) {
            // pairs, except the column the chain needs next (k+2): alone, and
            // first, so its projection k is out as early as possible
            if (chain && j != k + 2 && j + S < ncol) {
                update_pair(j, j + S, k);
                if (tid == 0) {
                    st_release(p.cflags + j, k + 1);
                    st_release(p.cflags + j + S, k + 1);
                }
                j += S;  // past the pair
                continue;
            }
            const bool ok = update_col(j, k, colp(j));
            // chain mode: column j has its first k+1 projections (an overflow
            // still reports progress: the chain's normalisation records it)
            if (chain && tid == 0) st_release(p.cflags + j, k + 1);
            if (p.trace && tid == 0 && j == k + 1) p.trace[(k + 1) * 8 + 1] = gtimer();
            if (ok && j == k + 1 && j < n) {
                if (!normalize_publish(j, colp(j))) {
                    abort = true;
                    break;
                }
            } else if (!ok && j == k + 1 && j < n) {
                if (tid == 0) {
                    __threadfence();
                    st_release(p.flags + j, 2);
                }
                abort = true;
                break;
            }
        }
        __syncthreads();
        if (p.trace && tid == 0) atomicMax(p.trace + (k + 1) * 8 + 3, gtimer());
    }

    // z = column_norm(b) by its owner (mgs.hpp:155)
    if (LSQ && !abort && bulk && (n % S) == own0) {
        R s = col_sq(colp(n));
        R z = rsqrt_ref(s);
        if (tid == 0) {
            if (!vfinite(s) || !vfinite(z)) record(1 + (long long)n * (ncol + 1), 0, XQR_OVERFLOW);
            store_real<L>(p.z, 1, z);
        }
    }
    if (!LSQ && chain) cg::this_grid().sync();  // the chain's published columns, visible to all
    if (!LSQ) {
        // Q = the normalised columns: planar -> AoS (L2 reads: in chain mode
        // another CTA wrote them)
        for (int j = c; j < n; j += G) {
            const double* src = colp(j);
            double* dst = p.q + (int64_t)j * m * L2;
            for (int e = tid; e < m * L2; e += kGridThreads) {
                const int plane = e % L2, i = e / L2;
                dst[e] = __ldcg(src + plane * f.LD + f.row_off(i));
            }
        }
    }
    cg::this_grid().sync();

    if (c == 0) {
        __shared__ unsigned long long s_key;
        if (tid == 0) s_key = __ldcg(p.key);
        if (p.trace && tid == 0) p.trace[n * 8 + 4] = p.trace[n * 8 + 5] = gtimer();
        __syncthreads();
        if (LSQ && s_key == kNoError) {
            // fused back substitution (mgs.hpp:157 -> :110-126); x in smem
            double* prep = p.rws + (int64_t)n * n * L2 + (int64_t)n * L2;
            bool bad = cta_back_substitute<L>(n, p.rws, ydst, smem, prep, &s_key,
                                              2 + (long long)n * (ncol + 1));
            if (!bad)
                for (int e = tid; e < n * L2; e += kGridThreads) p.x[e] = smem[e];
            __syncthreads();
            if (p.trace && tid == 0) p.trace[n * 8 + 6] = gtimer();
        }
        if (tid == 0) {
            unsigned long long key = s_key;
            xqr_status st;
            st.system = p.sys;
            st.code = key == kNoError ? 0 : (int)(key & 15);
            st.column = key == kNoError ? 0 : (int)((key >> 4) & 0xFFFFF);
            *p.st = st;
        }
    }
}

}  // namespace xb

namespace xb {

template <int L, bool LSQ>
cudaError_t launch_grid1(const GridParams& p, int grid, cudaStream_t s) {
    // rows per thread <= 4: a 3-level in-thread tree; 8 (m <= 2048): 4 levels
    auto kern = p.rpt <= 4 ? mgs_grid_kernel<L, 3, LSQ> : mgs_grid_kernel<L, 4, LSQ>;
    // the q_k staging area, plus (chain mode) the chain's two pivot-column buffers
    const size_t smem = sizeof(double) * 2 * L * kGridThreads * p.rpt * (p.chain ? 3 : 1);
    {  // (static + dynamic may pass 48 KB even when the dynamic part does not)
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    GridParams pp = p;
    void* args[] = {&pp};
    return cudaLaunchCooperativeKernel((const void*)kern, grid, kGridThreads, args, smem, s);
}

}  // namespace xb
