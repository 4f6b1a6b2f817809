// xbacksub.cuh -- CTA-level back substitution R x = y on the device.
//
// Reference: mgs.hpp:110-126 (column-oriented: x_k = x_k / r_kk by Smith
// division, complex.hpp:47-58, then x_j -= r_jk * x_k for every j < k).
// Every R-only part of the Smith division (the branch, t, the scaled
// denominator d and d's reciprocal prefix) is computed for all k in parallel
// first; the sequential sweep then runs only the dividend-dependent tail.
// Look-ahead: the owner of x_{k-1} divides it right after applying the x_k
// update, so each step costs a single CTA barrier.
#pragma once
#include "xcolumn.cuh"
#include "xqr_internal.h"

namespace xb {

// Quad-double t with every limb zero -- always so for MGS, whose diagonal is
// real: t = 0 / r_kk.  Then mul(x, t) (quad_double.hpp:267-338) is a
// function of the SIGN BITS of x alone for finite x: every partial product is
// a zero whose sign is the XOR of its factors' signs, every fma error term
// (x_i t_j) + (-p) is +0, and everything after adds and renormalises zeros.
// The 16 possible results (a sign nibble each) are computed once per pivot,
// off the sequential sweep, by mul itself on one representative per sign
// pattern, and the sweep then looks its product up instead of running a qd
// multiply whose renormalisation takes the reference's all-zero branch path.
XB_DEVICE int sign_nibble(const r4& x) {
    return (dbits(x.c0) < 0 ? 1 : 0) | (dbits(x.c1) < 0 ? 2 : 0) | (dbits(x.c2) < 0 ? 4 : 0) |
           (dbits(x.c3) < 0 ? 8 : 0);
}
XB_DEVICE r4 zeros_signed(int nib) {
    return {(nib & 1) ? -0.0 : 0.0, (nib & 2) ? -0.0 : 0.0, (nib & 4) ? -0.0 : 0.0, (nib & 8) ? -0.0 : 0.0};
}
XB_DEVICE bool all_zero(const r4& x) { return x.c0 == 0.0 && x.c1 == 0.0 && x.c2 == 0.0 && x.c3 == 0.0; }
XB_DEVICE bool all_finite(const r4& x) { return finite(x.c0) && finite(x.c1) && finite(x.c2) && finite(x.c3); }
// the table: nibble of mul(rep(pattern), t) at bits 4*pattern; ok = false if
// some product is not all zeros (then the table is not used)
XB_DEVICE unsigned long long zero_mul_table(const r4& t, bool& ok) {
    unsigned long long mask = 0;
    ok = true;
#pragma unroll 1
    for (int pat = 0; pat < 16; ++pat) {
        const r4 rep{(pat & 1) ? -1.0 : 1.0, (pat & 2) ? -0x1p-60 : 0x1p-60, (pat & 4) ? -0x1p-120 : 0x1p-120,
                     (pat & 8) ? -0x1p-180 : 0x1p-180};
        const r4 z = mul(rep, t);
        ok = ok && all_zero(z);
        mask |= (unsigned long long)sign_nibble(z) << (4 * pat);
    }
    return mask;
}

template <int L>
struct smith_prep {
    real_t<L> t, d;
    recip_t<real_t<L>> rc;
    int br;    // abs(d.re) >= abs(d.im)
    int code;  // error the division of x_k raises in the reference (0 = none)
    int zt = 0;                   // quad-double: t is all zeros, products from ztab
    unsigned long long ztab = 0;  // (zero_mul_table)
};
// x + z (either operand order) with z a qd of zeros equals x bit for bit
// when x is canonical: four non-zero finite limbs with fl(x_i + x_{i+1}) =
// x_i.  Walking the reference merge (quad_double.hpp:216-257): x's limbs
// come first (|x_i| > 0), each two_sum of adjacent limbs returns them
// unchanged, the two steps on x_2, x_3 emit x_0, x_1, the four steps on the
// zeros emit nothing (their error term is +0 whatever the zero's sign), the
// loop exit writes x_2, x_3, and renorm4 of a canonical tuple is the tuple.
XB_DEVICE bool qd_canonical(const r4& x) {
    return x.c0 != 0.0 && x.c1 != 0.0 && x.c2 != 0.0 && x.c3 != 0.0 && all_finite(x) &&
           dadd(x.c0, x.c1) == x.c0 && dadd(x.c1, x.c2) == x.c1 && dadd(x.c2, x.c3) == x.c2;
}

// mul(x, s.t) for the Smith numerator (complex.hpp:53/56), by the table when
// it applies (finite x; otherwise the multiply itself)
template <int L>
XB_DEVICE real_t<L> smith_tmul(const real_t<L>& x, const smith_prep<L>& s) {
    if constexpr (L == 4) {
        if (s.zt && all_finite(x)) return zeros_signed((int)(s.ztab >> (4 * sign_nibble(x))) & 15);
    }
    return mul(x, s.t);
}

// Store/load the prep record (3L+1 doubles) in global scratch.  Quad-double
// with zt: the table's 64 bits take t's head slot, t's sign bits go with the
// flags (t itself is zeros).
template <int L>
XB_DEVICE void prep_store(double* p, const smith_prep<L>& s) {
    store_real<L>(p, 1, s.t);
    store_real<L>(p + L, 1, s.d);
    if constexpr (L == 1) p[2] = s.rc.b;
    if constexpr (L == 2) store_real<2>(p + 2 * L, 1, s.rc.x1);
    if constexpr (L == 4) store_real<4>(p + 2 * L, 1, s.rc.x);
    int flags = s.br | (s.code << 4);
    if constexpr (L == 4) {
        if (s.zt) {
            flags |= (1 << 8) | (sign_nibble(s.t) << 9);
            p[0] = __longlong_as_double((long long)s.ztab);
        }
    }
    p[3 * L] = (double)flags;
}
template <int L>
XB_DEVICE smith_prep<L> prep_load(const double* p) {
    smith_prep<L> s;
    load_real<L>(p, 1, s.t);
    load_real<L>(p + L, 1, s.d);
    if constexpr (L == 1) s.rc.b = p[2];
    if constexpr (L == 2) load_real<2>(p + 2 * L, 1, s.rc.x1);
    if constexpr (L == 4) load_real<4>(p + 2 * L, 1, s.rc.x);
    int f = (int)p[3 * L];
    s.br = f & 15;
    s.code = (f >> 4) & 15;
    if constexpr (L == 4) {
        s.zt = (f >> 8) & 1;
        if (s.zt) {
            s.ztab = (unsigned long long)__double_as_longlong(p[0]);
            s.t = zeros_signed((f >> 9) & 15);
        }
    }
    return s;
}

template <int L>
XB_DEVICE cx<real_t<L>> load_aos(const double* p) {
    cx<real_t<L>> z;
    load_real<L>(p, 1, z.re);
    load_real<L>(p + L, 1, z.im);
    return z;
}
template <int L>
XB_DEVICE void store_aos(double* p, const cx<real_t<L>>& z) {
    store_real<L>(p, 1, z.re);
    store_real<L>(p + L, 1, z.im);
}

// x = Smith(xk / d) given the divisor-only prep (complex.hpp:50-57).
template <int L>
XB_DEVICE cx<real_t<L>> smith_apply(const cx<real_t<L>>& a, const smith_prep<L>& s) {
    using R = real_t<L>;
    rpair<R> p;
    if constexpr (L == 4) {
        if (s.zt) {
            p = {smith_tmul<L>(a.im, s), smith_tmul<L>(a.re, s)};
        } else {
            p = mul2(a.im, s.t, a.re, s.t);
        }
    } else {
        p = mul2(a.im, s.t, a.re, s.t);
    }
    rpair<R> nu = s.br ? add2(a.re, p.x, a.im, neg(p.y))    // a.re + a.im*t, a.im - a.re*t
                       : add2(p.y, a.im, p.x, neg(a.re));  // a.re*t + a.im, a.im*t - a.re
    return cdivide_real(cx<R>{nu.x, nu.y}, s.d, s.rc);
}

// CTA-wide.  r: AoS n x n (column-major), y: AoS n, xs: shared n*2L doubles,
// prep: global scratch n*(3L+1).  Records errors into *key (shared) with
// positions pos_base + (n-1-k).  Returns (uniformly) true on error.
// x = y; the R-only Smith prefix of every pivot, in parallel over the CTA.
// Errors found here are only *recorded in the prep*; they are raised when the
// sweep reaches step k, so an earlier-in-program-order failure still wins.
template <int L>
XB_DEVICE void cta_backsub_prep(int n, const double* r, const double* y, double* xs, double* prep) {
    using R = real_t<L>;
    using C = cx<R>;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int k = tid; k < n; k += nt) {
        store_aos<L>(xs + (size_t)k * 2 * L, load_aos<L>(y + (size_t)k * 2 * L));
        C d = load_aos<L>(r + ((size_t)k * n + k) * 2 * L);
        smith_prep<L> s;
        int dst = 0;
        if (is_zero(d.re) && is_zero(d.im)) {
            dst = 3;  // mgs.hpp:119-121 zero diagonal -> domain_error
            s.br = 1;
            s.t = d.re;
            s.d = d.re;
            int ignore = 0;
            s.rc = recip(rmake<R>(1.0), ignore);
        } else {
            s.br = ge(rabs(d.re), rabs(d.im)) ? 1 : 0;
            if (s.br) {
                s.t = rdiv(d.im, d.re, dst);
                s.d = add(d.re, mul(d.im, s.t));
            } else {
                s.t = rdiv(d.re, d.im, dst);
                s.d = add(mul(d.re, s.t), d.im);
            }
            if (!dst && (!vfinite(s.t) || !vfinite(s.d))) dst = 2;
            if (!dst) s.rc = recip(s.d, dst);
            if constexpr (L == 4) {
                if (!dst && all_zero(s.t)) {
                    bool ok = false;
                    s.ztab = zero_mul_table(s.t, ok);
                    s.zt = ok ? 1 : 0;
                }
            }
        }
        s.code = dst;
        prep_store<L>(prep + (size_t)k * (3 * L + 1), s);
    }
}

template <int L>
XB_DEVICE bool cta_back_substitute(int n, const double* r, const double* y, double* xs, double* prep,
                                unsigned long long* key, long long pos_base) {
    using R = real_t<L>;
    using C = cx<R>;
    const int tid = threadIdx.x, nt = blockDim.x;
    bool err = false;
    // x = y; R-only Smith prefix for every k in parallel.  Errors found here
    // are only *recorded in the prep*; they are raised when the sweep reaches
    // step k, so an earlier-in-program-order failure still wins.
    for (int k = tid; k < n; k += nt) {
        store_aos<L>(xs + (size_t)k * 2 * L, load_aos<L>(y + (size_t)k * 2 * L));
        C d = load_aos<L>(r + ((size_t)k * n + k) * 2 * L);
        smith_prep<L> s;
        int dst = 0;
        if (is_zero(d.re) && is_zero(d.im)) {
            dst = 3;  // mgs.hpp:119-121 zero diagonal -> domain_error
            s.br = 1;
            s.t = d.re;
            s.d = d.re;
            int ignore = 0;
            s.rc = recip(rmake<R>(1.0), ignore);
        } else {
            s.br = ge(rabs(d.re), rabs(d.im)) ? 1 : 0;
            if (s.br) {
                s.t = rdiv(d.im, d.re, dst);
                s.d = add(d.re, mul(d.im, s.t));
            } else {
                s.t = rdiv(d.re, d.im, dst);
                s.d = add(mul(d.re, s.t), d.im);
            }
            if (!dst && (!vfinite(s.t) || !vfinite(s.d))) dst = 2;
            if (!dst) s.rc = recip(s.d, dst);
        }
        s.code = dst;
        prep_store<L>(prep + (size_t)k * (3 * L + 1), s);
    }
    __syncthreads();
    // last unknown
    if (tid == (n - 1) % nt) {
        smith_prep<L> s = prep_load<L>(prep + (size_t)(n - 1) * (3 * L + 1));
        C xk = load_aos<L>(xs + (size_t)(n - 1) * 2 * L);
        if (s.code) {
            atomicMin(key, status_key(pos_base, 0, s.code));
            err = true;
        } else {
            xk = smith_apply<L>(xk, s);
            if (!cfinite(xk)) {
                atomicMin(key, status_key(pos_base, 0, 2));
                err = true;
            }
        }
        store_aos<L>(xs + (size_t)(n - 1) * 2 * L, xk);
    }
    if (__syncthreads_or(err)) return true;
    if (n <= nt) {
        // one unknown per thread: x_j stays in registers and r_{j,k-1} is
        // read ahead during step k, so the step is the arithmetic + a barrier
        const int j = tid;
        C xj{}, rn{};
        if (j < n) xj = load_aos<L>(xs + (size_t)j * 2 * L);
        if (j < n - 1) rn = load_aos<L>(r + ((size_t)(n - 1) * n + j) * 2 * L);
        for (int k = n - 1; k >= 1; --k) {
            const C xk = load_aos<L>(xs + (size_t)k * 2 * L);
            const C rc = rn;
            if (j < k - 1) rn = load_aos<L>(r + ((size_t)(k - 1) * n + j) * 2 * L);
            if (j < k) {
                xj = csub(xj, cmul(rc, xk));
                if (!cfinite(xj)) {
                    atomicMin(key, status_key(pos_base + (n - 1 - k), 0, 2));
                    err = true;
                } else if (j == k - 1) {
                    smith_prep<L> s = prep_load<L>(prep + (size_t)j * (3 * L + 1));
                    if (s.code) {
                        atomicMin(key, status_key(pos_base + (n - k), 0, s.code));
                        err = true;
                    } else {
                        xj = smith_apply<L>(xj, s);
                        if (!cfinite(xj)) {
                            atomicMin(key, status_key(pos_base + (n - k), 0, 2));
                            err = true;
                        }
                    }
                }
                if (j == k - 1) store_aos<L>(xs + (size_t)j * 2 * L, xj);  // final: the next steps read it
            }
            if (__syncthreads_or(err)) return true;
        }
        return false;
    }
    for (int k = n - 1; k >= 1; --k) {
        const C xk = load_aos<L>(xs + (size_t)k * 2 * L);
        const double* rk = r + (size_t)k * n * 2 * L;
        for (int j = tid; j < k; j += nt) {
            C xj = load_aos<L>(xs + (size_t)j * 2 * L);
            xj = csub(xj, cmul(load_aos<L>(rk + (size_t)j * 2 * L), xk));
            if (!cfinite(xj)) {
                atomicMin(key, status_key(pos_base + (n - 1 - k), 0, 2));
                err = true;
            } else if (j == k - 1) {
                smith_prep<L> s = prep_load<L>(prep + (size_t)j * (3 * L + 1));
                if (s.code) {
                    atomicMin(key, status_key(pos_base + (n - k), 0, s.code));
                    err = true;
                } else {
                    xj = smith_apply<L>(xj, s);
                    if (!cfinite(xj)) {
                        atomicMin(key, status_key(pos_base + (n - k), 0, 2));
                        err = true;
                    }
                }
            }
            store_aos<L>(xs + (size_t)j * 2 * L, xj);
        }
        if (__syncthreads_or(err)) return true;
    }
    return false;
}

// Warp-specialised back substitution of one system (mgs.hpp:117-124): a
// LANE PAIR owns an unknown and splits every complex operation into its real
// half (even lane) and imaginary half (odd lane) -- the halves of cmul / csub
// / the Smith quotient are independent (complex.hpp:41-58) -- and there is no
// CTA barrier per step.  The sequential chain of the column sweep is
//   x_k final -> x_{k-1} -= r_{k-1,k} x_k -> Smith division of x_{k-1},
// and every other update x_j -= r_jk x_k (j <= k-2) can run a step or more
// behind it.  So:
//   * warp 0 is the FINISHER: its lane pair 0 applies the last update to
//     x_{k-1}, divides it, keeps it in registers for the next step and
//     publishes it (shared memory + a monotone `frontier`);
//   * warps 1..NW-1 are UPDATERS: unknowns are dealt to them in blocks of 16
//     (one per lane pair); for every published x_k, in order, an updater
//     applies x_j -= r_jk x_k to its own j <= k-2, highest block first, and
//     advances its `hi` mark after that block -- what the finisher waits for
//     before taking x_{k-1}.  Slots past the other warps' go to the warps on
//     the finisher's SMSP (XB_BS_ISOLATE 2), which stay idle for n <= 16 NR.
// Nothing on the chain waits for a CTA barrier or for another pair's
// data-dependent (divergent) add paths; R is read ahead into registers.
//
// Errors (the reference raises the first in program order): a failing
// divide of x_k or update at step k records its status key and raises
// `stop` to k; a warp stops before any step k <= stop, so every step above
// the first failure is completed by every warp and the minimum key is the
// reference's.  xs (n*2L doubles), prep (n*(3L+1)) and sync (2 + NW ints)
// are shared memory; blockDim.x is a multiple of 32, at least 64.  Returns
// (uniformly) true on error.
#ifndef XB_BS_ISOLATE
#define XB_BS_ISOLATE 2
#endif
// CTA-scope flag handoff in shared memory: an acquire load is a plain LDS on
// sm_100a (no fence); a release store costs one MEMBAR.ALL.CTA, lighter than
// the MEMBAR.SC.CTA that __threadfence_block() emits
XB_DEVICE int bs_acquire(const volatile int* f) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];"
                 : "=r"(v)
                 : "r"((unsigned)__cvta_generic_to_shared((const void*)f))
                 : "memory");
    return v;
}
XB_DEVICE void bs_release(volatile int* f, int v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared((void*)f)), "r"(v)
                 : "memory");
}
template <int L>
XB_DEVICE bool flow_back_substitute(int n, const double* r, const double* y, double* xs, double* prep,
                                    int* sync, unsigned long long* key, long long pos_base,
                                    unsigned long long* trace = nullptr) {
    using R = real_t<L>;
    constexpr unsigned kFull = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
    // XB_BS_ISOLATE: the warps sharing the finisher's SM sub-partition (warp
    // id = 0 mod 4) stay idle, so the sequential chain does not compete for
    // that SMSP's FP64 issue; updater u runs on warp u + 1 + u / 3
#if XB_BS_ISOLATE == 2
    // ... until every other warp holds a block: the idle ones then take the
    // next slots (16 * (NW - 1) unknowns per sweep)
    const int NR = NW - (NW + 3) / 4;  // updaters off the finisher's SMSP
    const int NU = NW - 1;
    const bool updater = warp > 0;
    const int uo = (warp & 3) ? warp - 1 - (warp >> 2) : NR + (warp >> 2) - 1;
    auto uwarp = [NR](int u) { return u < NR ? u + 1 + u / 3 : 4 * (u - NR + 1); };
#elif XB_BS_ISOLATE
    const int NU = NW - (NW + 3) / 4;
    const bool updater = warp > 0 && (warp & 3) != 0;
    const int uo = warp - 1 - (warp >> 2);
    auto uwarp = [](int u) { return u + 1 + u / 3; };
#else
    const int NU = NW - 1;
    const bool updater = warp > 0;
    const int uo = warp - 1;
    auto uwarp = [](int u) { return u + 1; };
#endif
    const int part = lane & 1, pl = lane >> 1, BW = 16 * NU;
    const unsigned pmask = 3u << (lane & 30);
    volatile int* frontier = sync;  // lowest k whose x_k is final and in xs
    volatile int* stop = sync + 1;  // highest step at which an error occurred
    // hi[w]: updater w applied every x_k, k > hi[w], to all its unknowns and
    // x_{hi[w]} to its highest block (which holds the finisher's next unknown)
    volatile int* hi = sync + 2;
    cta_backsub_prep<L>(n, r, y, xs, prep);
    if (tid == 0) {
        sync[0] = n;
        sync[1] = -1;
    }
    if (tid < NW) sync[2 + tid] = n;
    __syncthreads();
    bool err = false;
    auto fail = [&](int step, int code) {
        if (part == 0) {
            atomicMin(key, status_key(pos_base + (n - 1 - step), 0, code));
            atomicMax((int*)stop, step);
        }
        err = true;
    };
    auto xs_part = [&](int j, int pp) { return xs + (size_t)j * 2 * L + pp * L; };
    auto rpart = [&](int j, int k, int pp) { return r + ((size_t)k * n + j) * 2 * L + pp * L; };
    // own half of Smith(x / d_j) (complex.hpp:50-57), R-only parts from prep
    auto smith = [&](const R& are, const R& aim, int j, int& code) -> R {
        const smith_prep<L> sp = prep_load<L>(prep + (size_t)j * (3 * L + 1));
        code = sp.code;
        R num;
        // (a zero product added to a canonical x leaves x: qd_canonical)
        if (sp.br) {
            const R x = part ? aim : are;
            const R prod = smith_tmul<L>(part ? are : aim, sp);
            bool keep = false;
            if constexpr (L == 4) keep = sp.zt && all_zero(prod) && qd_canonical(x);
            num = keep ? x : add(x, part ? neg(prod) : prod);
        } else {
            const R x = part ? neg(are) : aim;
            const R prod = smith_tmul<L>(part ? aim : are, sp);
            bool keep = false;
            if constexpr (L == 4) keep = sp.zt && all_zero(prod) && qd_canonical(x);
            num = keep ? x : add(prod, x);
        }
        return divide_inline(num, sp.d, sp.rc);
    };
    // own half of x_j - r_jk x_k (cmul complex.hpp:41-44, csub :31-34), given
    // this lane's (y1, y2) = (x_k.re, x_k.im) or (x_k.im, x_k.re)
    auto update = [&](const R& xj, const R& rre, const R& rim, const R& y1, const R& y2) -> R {
        rpair<R> pr = mul2(rre, y1, rim, y2);
        return sub(xj, add(pr.x, part ? pr.y : neg(pr.y)));
    };

    if (warp == 0) {
        // ---------------- finisher ----------------
        if (lane < 2) {
            int code = 0;
            R are, aim;
            load_real<L>(xs_part(n - 1, 0), 1, are);
            load_real<L>(xs_part(n - 1, 1), 1, aim);
            R v = smith(are, aim, n - 1, code);  // x_{n-1} = y_{n-1} / r_{n-1,n-1}
            if (code) {
                fail(n - 1, code);
            } else if (!vfinite(v) || !vfinite(shfl_pair(v, pmask))) {
                fail(n - 1, 2);
            }
            R rre, rim;  // r_{k-1,k} for the next step, read ahead
            if (n >= 2) {
                load_real<L>(rpart(n - 2, n - 1, 0), 1, rre);
                load_real<L>(rpart(n - 2, n - 1, 1), 1, rim);
            }
            store_real<L>(xs_part(n - 1, part), 1, v);
            __syncwarp(3u);
            if (lane == 0) {
                bs_release(frontier, n - 1);
            }
            // owner (updater index) of x_{k-1}, stepped down with k: no division on the chain
            int ublk = n >= 2 ? ((n - 2) >> 4) % NU : 0;
            for (int k = n - 1; k >= 1 && !err; --k) {
                // dev instrumentation (XQR_GRID_TRACE): SM cycles per phase
                unsigned long long c0 = trace ? clock64() : 0;
                // x_{k-1} has every update but x_k's once its updater is past k+1
                const int w = uwarp(ublk);
                if (((k - 1) & 15) == 0) ublk = ublk ? ublk - 1 : NU - 1;
                int spins = 0;
                while (bs_acquire(&hi[w]) > k + 1 && bs_acquire(stop) < k) {
                    __nanosleep(20);
                    ++spins;
                }
                unsigned long long c1 = trace ? clock64() : 0, c2 = 0;
                if (*stop >= k) break;
                // (y1, y2) = (own half, other half) of x_k
                const R y1 = v, y2 = shfl_pair(v, 3u);
                R xj;
                load_real<L>(xs_part(k - 1, part), 1, xj);
                const R cr = rre, ci = rim;
                if (k >= 2) {  // read ahead r_{k-2,k-1}
                    load_real<L>(rpart(k - 2, k - 1, 0), 1, rre);
                    load_real<L>(rpart(k - 2, k - 1, 1), 1, rim);
                }
                v = update(xj, cr, ci, y1, y2);
                if (!vfinite(v) || !vfinite(shfl_pair(v, 3u))) {
                    fail(k, 2);
                } else {
                    if (trace) c2 = clock64();
                    const R ov = shfl_pair(v, 3u);
                    v = smith(part ? ov : v, part ? v : ov, k - 1, code);
                    if (code) {
                        fail(k - 1, code);
                    } else if (!vfinite(v) || !vfinite(shfl_pair(v, 3u))) {
                        fail(k - 1, 2);
                    }
                }
                unsigned long long c3 = trace ? clock64() : 0;
                store_real<L>(xs_part(k - 1, part), 1, v);
                __syncwarp(3u);
                if (lane == 0) {
                    bs_release(frontier, k - 1);
                }
                if (trace && lane == 0) {
                    trace[8 * k + 0] = c0;
                    trace[8 * k + 1] = c1;
                    trace[8 * k + 2] = c2;
                    trace[8 * k + 3] = c3;
                    trace[8 * k + 4] = clock64();
                    trace[8 * k + 7] = spins;
                }
            }
        }
    } else if (updater) {
        // ---------------- updaters ----------------
        const int base = 16 * uo + pl;  // this pair's lowest unknown
        int k = n - 1;
        for (; k >= 2; --k) {
            if (16 * uo > k - 2) break;  // every own unknown is past its updates
            if (lane == 0) {
                while (bs_acquire(frontier) > k && bs_acquire(stop) < k) __nanosleep(32);
            }
            __syncwarp();  // orders lane 0's acquire before the warp's reads
            if (__any_sync(kFull, *stop >= k)) break;
            // dev instrumentation: the finisher's next input (x_{k-2}) taken / done
            const bool crit = trace && lane == 0 && uwarp(((k - 2) >> 4) % NU) == warp;
            if (crit) trace[8 * (k - 1) + 5] = clock64();
            R xkre, xkim;
            load_real<L>(xs_part(k, 0), 1, xkre);
            load_real<L>(xs_part(k, 1), 1, xkim);
            const R y1 = part ? xkim : xkre, y2 = part ? xkre : xkim;
            // highest own j <= k-2 first: the finisher needs x_{k-2} next --
            // and may take it as soon as this warp's highest block is done
            // (`hi`), before the lower blocks
            const int j0 = base <= k - 2 ? base + ((k - 2 - base) / BW) * BW : -1;
            auto upd = [&](int j) {
                R rre, rim, xj;
                load_real<L>(rpart(j, k, 0), 1, rre);
                load_real<L>(rpart(j, k, 1), 1, rim);
                load_real<L>(xs_part(j, part), 1, xj);
                const R v = update(xj, rre, rim, y1, y2);
                if (!vfinite(v) || !vfinite(shfl_pair(v, pmask))) fail(k, 2);
                store_real<L>(xs_part(j, part), 1, v);
            };
#ifndef XB_BS_EXPERIMENT
            if (j0 >= 0) upd(j0);
            __syncwarp();
            if (lane == 0) {
                bs_release(&hi[warp], k);
                if (crit) trace[8 * (k - 1) + 6] = clock64();
            }
            for (int j = j0 - BW; j >= 0; j -= BW) upd(j);
#endif
            // R is known from the start: pull next step's r_{j,k-1} into L1
            for (int j = base <= k - 3 ? base + ((k - 3 - base) / BW) * BW : -1; j >= 0; j -= BW)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(rpart(j, k - 1, part)));
        }
        __syncwarp();
        if (lane == 0 && k < 2) hi[warp] = -1;  // nothing left: never hold the finisher
        if (lane == 0 && k >= 2 && 16 * uo > k - 2) hi[warp] = -1;
    }
    return __syncthreads_or(err);
}

}  // namespace xb
