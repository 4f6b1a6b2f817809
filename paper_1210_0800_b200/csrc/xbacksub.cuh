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

}  // namespace xb
