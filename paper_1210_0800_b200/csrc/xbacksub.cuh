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

template <int L>
struct smith_prep {
    real_t<L> t, d;
    recip_t<real_t<L>> rc;
    int br;    // abs(d.re) >= abs(d.im)
    int code;  // error the division of x_k raises in the reference (0 = none)
};

// Store/load the prep record (3L+1 doubles) in global scratch.
template <int L>
XB_DEVICE void prep_store(double* p, const smith_prep<L>& s) {
    store_real<L>(p, 1, s.t);
    store_real<L>(p + L, 1, s.d);
    if constexpr (L == 1) p[2] = s.rc.b;
    if constexpr (L == 2) store_real<2>(p + 2 * L, 1, s.rc.x1);
    if constexpr (L == 4) store_real<4>(p + 2 * L, 1, s.rc.x);
    p[3 * L] = (double)(s.br | (s.code << 4));
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
    s.code = f >> 4;
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
    rpair<R> p = mul2(a.im, s.t, a.re, s.t);
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
            if (!dst && (!finite(head(s.t)) || !finite(head(s.d)))) dst = 2;
            if (!dst) s.rc = recip(s.d, dst);
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
            if (!dst && (!finite(head(s.t)) || !finite(head(s.d)))) dst = 2;
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

// Latency-first form for the single-system quad-double kernel (xgrid2.cuh):
// a LANE PAIR owns unknowns j = pair, pair + P, ... (P = blockDim.x / 2) and
// splits every complex operation into its real half (even lane) and
// imaginary half (odd lane) -- the halves of cmul / csub / the Smith
// quotient are independent (complex.hpp:41-58).  Per step k
// (mgs.hpp:117-124): x_j -= r_jk * x_k for j < k, the owner of k-1 first, and
// the owner of x_{k-1} divides it at once (look-ahead).  R-only Smith parts
// come from cta_backsub_prep.  Same operations, operands and order as the
// reference; returns (uniformly) true on error.
template <int L>
XB_DEVICE bool pair_back_substitute(int n, const double* r, const double* y, double* xs, double* prep,
                                    unsigned long long* key, long long pos_base) {
    using R = real_t<L>;
    const int tid = threadIdx.x, P = blockDim.x / 2, pair = tid >> 1, part = tid & 1;
    const unsigned pmask = 3u << (tid & 30);  // this lane pair
    cta_backsub_prep<L>(n, r, y, xs, prep);
    __syncthreads();
    bool err = false;
    // own half of x_j = x_j / d_j (complex.hpp:50-57) given both halves of x_j
    auto smith = [&](const R& are, const R& aim, int j) -> R {
        const smith_prep<L> sp = prep_load<L>(prep + (size_t)j * (3 * L + 1));
        R num;
        if (sp.br) {  // a.re + a.im*t  |  a.im - a.re*t
            const R prod = mul(part ? are : aim, sp.t);
            num = add(part ? aim : are, part ? neg(prod) : prod);
        } else {      // a.re*t + a.im  |  a.im*t - a.re
            const R prod = mul(part ? aim : are, sp.t);
            num = add(prod, part ? neg(are) : aim);
        }
        return divide(num, sp.d, sp.rc);
    };
    auto xs_part = [&](int j, int pp) { return xs + (size_t)j * 2 * L + pp * L; };
    // last unknown
    if (pair == (n - 1) % P) {
        const smith_prep<L> sp = prep_load<L>(prep + (size_t)(n - 1) * (3 * L + 1));
        R are, aim;
        load_real<L>(xs_part(n - 1, 0), 1, are);
        load_real<L>(xs_part(n - 1, 1), 1, aim);
        R v = part ? aim : are;
        if (sp.code) {
            if (part == 0) atomicMin(key, status_key(pos_base, 0, sp.code));
            err = true;
        } else {
            v = smith(are, aim, n - 1);
            if (!finite(head(v)) || !finite(head(shfl_pair(v, pmask)))) {
                if (part == 0) atomicMin(key, status_key(pos_base, 0, 2));
                err = true;
            }
        }
        store_real<L>(xs_part(n - 1, part), 1, v);
    }
    if (__syncthreads_or(err)) return true;
    for (int k = n - 1; k >= 1; --k) {
        R xkre, xkim;
        load_real<L>(xs_part(k, 0), 1, xkre);
        load_real<L>(xs_part(k, 1), 1, xkim);
        const double* rk = r + (size_t)k * n * 2 * L;
        // highest owned j < k first: the owner of k-1 reaches its division soonest
        int j = pair + ((k - 1 - pair) / P) * P;
        if (k - 1 < pair) j = -1;
        for (; j >= 0; j -= P) {
            R rre, rim, xj;
            load_real<L>(rk + (size_t)j * 2 * L, 1, rre);
            load_real<L>(rk + (size_t)j * 2 * L + L, 1, rim);
            load_real<L>(xs_part(j, part), 1, xj);
            // t = cmul(r_jk, x_k) (complex.hpp:41-44): own half
            const R y1 = part ? xkim : xkre, y2 = part ? xkre : xkim;
            rpair<R> pr = mul2(rre, y1, rim, y2);
            const R t = add(pr.x, part ? pr.y : neg(pr.y));
            R v = sub(xj, t);  // csub (complex.hpp:31-34)
            bool bad = !finite(head(v)) || !finite(head(shfl_pair(v, pmask)));
            if (bad) {
                if (part == 0) atomicMin(key, status_key(pos_base + (n - 1 - k), 0, 2));
                err = true;
            } else if (j == k - 1) {
                const smith_prep<L> sp = prep_load<L>(prep + (size_t)j * (3 * L + 1));
                if (sp.code) {
                    if (part == 0) atomicMin(key, status_key(pos_base + (n - k), 0, sp.code));
                    err = true;
                } else {
                    const R o = shfl_pair(v, pmask);
                    v = smith(part ? o : v, part ? v : o, j);
                    if (!finite(head(v)) || !finite(head(shfl_pair(v, pmask)))) {
                        if (part == 0) atomicMin(key, status_key(pos_base + (n - k), 0, 2));
                        err = true;
                    }
                }
            }
            store_real<L>(xs_part(j, part), 1, v);
        }
        // R is known from the start: pull next step's r_{j,k-1} (and the
        // next pivot's Smith record) into L1 while the barrier drains
        if (k >= 2) {
            const double* rn = r + (size_t)(k - 1) * n * 2 * L;
            for (int jj = pair; jj < k - 1; jj += P)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(rn + (size_t)jj * 2 * L + part * L));
            if (tid == 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(prep + (size_t)(k - 2) * (3 * L + 1)));
        }
        if (__syncthreads_or(err)) return true;
    }
    return false;
}

}  // namespace xb
