/*
 * xqr_oracle_tmpl.h -- CPU ORACLE (test infrastructure only).
 * Complex arithmetic, the fixed reduction tree and the MGS algorithms,
 * restated from complex.hpp / reduction.hpp / mgs.hpp.  Included once per
 * real type with:
 *   R        real struct (xo_d / xo_dd / xo_qd)
 *   RP(x)    prefix for the real ops (xo_dd_##x ...)
 *   CP(x)    prefix for the functions this file defines
 *   LIMBS    1, 2 or 4
 *   EPSILON  real_traits<R>::epsilon (real_type.hpp:33-47)
 */

typedef struct {
    R re, im;
} CP(cplx);

static inline R CP(rzero)(void) {
    R z;
    memset(&z, 0, sizeof z);
    return z;
}
static inline R CP(rfrom)(double v) {
    R z = CP(rzero)();
    ((double*)&z)[0] = v;
    return z;
}
static inline CP(cplx) CP(load)(const double* p) {
    CP(cplx) z;
    memcpy(&z.re, p, sizeof(R));
    memcpy(&z.im, p + LIMBS, sizeof(R));
    return z;
}
static inline void CP(store)(double* p, CP(cplx) z) {
    memcpy(p, &z.re, sizeof(R));
    memcpy(p + LIMBS, &z.im, sizeof(R));
}

/* complex.hpp:21-24 */
static inline CP(cplx) CP(conj)(CP(cplx) z) {
    CP(cplx) r = {z.re, RP(neg)(z.im)};
    return r;
}
/* complex.hpp:26-29 */
static inline CP(cplx) CP(add)(CP(cplx) a, CP(cplx) b) {
    CP(cplx) r = {RP(add)(a.re, b.re), RP(add)(a.im, b.im)};
    return r;
}
/* complex.hpp:31-34 */
static inline CP(cplx) CP(sub)(CP(cplx) a, CP(cplx) b) {
    CP(cplx) r = {RP(sub)(a.re, b.re), RP(sub)(a.im, b.im)};
    return r;
}
/* complex.hpp:41-44 */
static inline CP(cplx) CP(mul)(CP(cplx) a, CP(cplx) b) {
    R rr = RP(mul)(a.re, b.re);
    R ii = RP(mul)(a.im, b.im);
    R ri = RP(mul)(a.re, b.im);
    R ir = RP(mul)(a.im, b.re);
    CP(cplx) r = {RP(sub)(rr, ii), RP(add)(ri, ir)};
    return r;
}
/* complex.hpp:47-58 (Smith) */
static inline CP(cplx) CP(div)(CP(cplx) a, CP(cplx) b) {
    R zero = CP(rzero)();
    if (RP(eq)(b.re, zero) && RP(eq)(b.im, zero)) xo_throw(XO_DOMAIN, 0);
    R abs_re = RP(abs)(b.re), abs_im = RP(abs)(b.im);
    if (RP(ge)(abs_re, abs_im)) {
        R t = RP(div)(b.im, b.re);
        R d = RP(add)(b.re, RP(mul)(b.im, t));
        CP(cplx) r = {RP(div)(RP(add)(a.re, RP(mul)(a.im, t)), d),
                      RP(div)(RP(sub)(a.im, RP(mul)(a.re, t)), d)};
        return r;
    }
    R t = RP(div)(b.re, b.im);
    R d = RP(add)(RP(mul)(b.re, t), b.im);
    CP(cplx) r = {RP(div)(RP(add)(RP(mul)(a.re, t), a.im), d),
                  RP(div)(RP(sub)(RP(mul)(a.im, t), a.re), d)};
    return r;
}
/* complex.hpp:61-65 */
static inline CP(cplx) CP(div_real)(CP(cplx) a, R r) {
    if (RP(eq)(r, CP(rzero)())) xo_throw(XO_DOMAIN, 0);
    CP(cplx) o = {RP(div)(a.re, r), RP(div)(a.im, r)};
    return o;
}
/* complex.hpp:77-85 */
static inline R CP(abs2)(CP(cplx) z) { return RP(add)(RP(mul)(z.re, z.re), RP(mul)(z.im, z.im)); }
static inline R CP(cabs)(CP(cplx) z) { return RP(sqrt)(CP(abs2)(z)); }

/* reduction.hpp:34-40 */
static CP(cplx) CP(tree_reduce)(CP(cplx)* t, int64_t len) {
    if (len == 0) {
        CP(cplx) z = {CP(rzero)(), CP(rzero)()};
        return z;
    }
    for (int64_t stride = 1; stride < len; stride <<= 1)
        for (int64_t i = 0; i + stride < len; i += 2 * stride) t[i] = CP(add)(t[i], t[i + stride]);
    return t[0];
}
/* reduction.hpp:45-51 */
static CP(cplx) CP(tree_inner_product)(const CP(cplx)* x, const CP(cplx)* y, int64_t len,
                                       CP(cplx)* scratch) {
    for (int64_t l = 0; l < len; ++l) scratch[l] = CP(mul)(CP(conj)(x[l]), y[l]);
    return CP(tree_reduce)(scratch, len);
}

/* mgs.hpp:38-42 */
static R CP(column_norm)(const CP(cplx)* a, int64_t m, CP(cplx)* scratch) {
    CP(cplx) s = CP(tree_inner_product)(a, a, m, scratch);
    return RP(sqrt)(s.re);
}
/* mgs.hpp:46-53 */
static R CP(normalize_column)(CP(cplx)* a, int64_t m, CP(cplx)* scratch, R threshold,
                              int column_index) {
    R rkk = CP(column_norm)(a, m, scratch);
    if (RP(le)(rkk, threshold)) xo_throw(XO_BREAKDOWN, column_index);
    for (int64_t i = 0; i < m; ++i) a[i] = CP(div_real)(a[i], rkk);
    return rkk;
}
/* mgs.hpp:57-61 */
static CP(cplx) CP(remove_projection)(const CP(cplx)* q, CP(cplx)* a, int64_t m,
                                      CP(cplx)* scratch) {
    CP(cplx) r = CP(tree_inner_product)(q, a, m, scratch);
    for (int64_t i = 0; i < m; ++i) a[i] = CP(sub)(a[i], CP(mul)(r, q[i]));
    return r;
}
/* mgs.hpp:66-70 */
static R CP(breakdown_threshold)(int64_t rows, R max_column_norm) {
    double scale = (double)rows * EPSILON;
    return RP(mul)(CP(rfrom)(scale), max_column_norm);
}

static void CP(load_cols)(CP(cplx)* cols, const double* a, int64_t m, int64_t n) {
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) cols[j * m + i] = CP(load)(a + (j * m + i) * 2 * LIMBS);
}

/* mgs.hpp:84-106 */
static void CP(mgs_qr)(int64_t m, int64_t n, const double* a, double* qout, double* rout) {
    CP(cplx)* cols = (CP(cplx)*)malloc(sizeof(CP(cplx)) * (size_t)(m * n));
    CP(cplx)* scratch = (CP(cplx)*)malloc(sizeof(CP(cplx)) * (size_t)m);
    CP(cplx)* rr = (CP(cplx)*)calloc((size_t)(n * n), sizeof(CP(cplx)));
    CP(load_cols)(cols, a, m, n);

    R max_norm = CP(rzero)();
    for (int64_t j = 0; j < n; ++j) {
        R nrm = CP(column_norm)(cols + j * m, m, scratch);
        if (RP(lt)(max_norm, nrm)) max_norm = nrm;
    }
    R threshold = CP(breakdown_threshold)(m, max_norm);

    for (int64_t k = 0; k < n; ++k) {
        R rkk = CP(normalize_column)(cols + k * m, m, scratch, threshold, (int)(k + 1));
        CP(cplx) d = {rkk, CP(rzero)()};
        rr[k * n + k] = d;
        for (int64_t j = k + 1; j < n; ++j)
            rr[j * n + k] = CP(remove_projection)(cols + k * m, cols + j * m, m, scratch);
    }
    for (int64_t e = 0; e < m * n; ++e) CP(store)(qout + e * 2 * LIMBS, cols[e]);
    for (int64_t e = 0; e < n * n; ++e) CP(store)(rout + e * 2 * LIMBS, rr[e]);
    free(cols);
    free(scratch);
    free(rr);
}

/* mgs.hpp:110-126 (r: n x n column-major, y, x: n) */
static void CP(back_substitute_cols)(int64_t n, const CP(cplx)* r, const CP(cplx)* y,
                                     CP(cplx)* x) {
    R zero = CP(rzero)();
    for (int64_t i = 0; i < n; ++i) x[i] = y[i];
    for (int64_t k = n; k-- > 0;) {
        CP(cplx) d = r[k * n + k];
        if (RP(eq)(d.re, zero) && RP(eq)(d.im, zero)) xo_throw(XO_DOMAIN, 0);
        x[k] = CP(div)(x[k], d);
        for (int64_t j = 0; j < k; ++j) x[j] = CP(sub)(x[j], CP(mul)(r[k * n + j], x[k]));
    }
}

static void CP(back_substitute)(int64_t n, const double* r, const double* y, double* xout) {
    CP(cplx)* rr = (CP(cplx)*)malloc(sizeof(CP(cplx)) * (size_t)(n * n));
    CP(cplx)* yy = (CP(cplx)*)malloc(sizeof(CP(cplx)) * (size_t)n);
    CP(cplx)* xx = (CP(cplx)*)malloc(sizeof(CP(cplx)) * (size_t)n);
    CP(load_cols)(rr, r, n, n);
    CP(load_cols)(yy, y, n, 1);
    CP(back_substitute_cols)(n, rr, yy, xx);
    for (int64_t e = 0; e < n; ++e) CP(store)(xout + e * 2 * LIMBS, xx[e]);
    free(rr);
    free(yy);
    free(xx);
}

/* mgs.hpp:131-158 */
static void CP(lsq_solve)(int64_t m, int64_t n, const double* a, const double* b, double* xout,
                          double* zout) {
    CP(cplx)* cols = (CP(cplx)*)malloc(sizeof(CP(cplx)) * (size_t)(m * (n + 1)));
    CP(cplx)* scratch = (CP(cplx)*)malloc(sizeof(CP(cplx)) * (size_t)m);
    CP(cplx)* rr = (CP(cplx)*)calloc((size_t)(n * n), sizeof(CP(cplx)));
    CP(cplx)* y = (CP(cplx)*)calloc((size_t)n, sizeof(CP(cplx)));
    CP(cplx)* x = (CP(cplx)*)calloc((size_t)n, sizeof(CP(cplx)));
    CP(load_cols)(cols, a, m, n);
    CP(load_cols)(cols + n * m, b, m, 1);

    /* mgs.hpp:72-80 max_column_norm over the n+1 columns */
    R max_norm = CP(rzero)();
    for (int64_t j = 0; j <= n; ++j) {
        R nrm = CP(column_norm)(cols + j * m, m, scratch);
        if (RP(lt)(max_norm, nrm)) max_norm = nrm;
    }
    R threshold = CP(breakdown_threshold)(m, max_norm);

    for (int64_t k = 0; k < n; ++k) {
        R rkk = CP(normalize_column)(cols + k * m, m, scratch, threshold, (int)(k + 1));
        CP(cplx) d = {rkk, CP(rzero)()};
        rr[k * n + k] = d;
        for (int64_t j = k + 1; j < n; ++j)
            rr[j * n + k] = CP(remove_projection)(cols + k * m, cols + j * m, m, scratch);
        y[k] = CP(remove_projection)(cols + k * m, cols + n * m, m, scratch);
    }
    R z = CP(column_norm)(cols + n * m, m, scratch);
    CP(back_substitute_cols)(n, rr, y, x);
    for (int64_t e = 0; e < n; ++e) CP(store)(xout + e * 2 * LIMBS, x[e]);
    memcpy(zout, &z, sizeof(R));
    free(cols);
    free(scratch);
    free(rr);
    free(y);
    free(x);
}

/* mgs.hpp:161-178 */
static void CP(residual_max_entry)(int64_t m, int64_t n, const double* a, const double* q,
                                   const double* r, double* out) {
    R worst = CP(rzero)();
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t i = 0; i < m; ++i) {
            CP(cplx) s = {CP(rzero)(), CP(rzero)()};
            for (int64_t l = 0; l <= j; ++l)
                s = CP(add)(s, CP(mul)(CP(load)(q + (l * m + i) * 2 * LIMBS),
                                       CP(load)(r + (j * n + l) * 2 * LIMBS)));
            R e = CP(cabs)(CP(sub)(CP(load)(a + (j * m + i) * 2 * LIMBS), s));
            if (RP(lt)(worst, e)) worst = e;
        }
    }
    memcpy(out, &worst, sizeof(R));
}

/* mgs.hpp:208-222 */
static void CP(orthogonality_defect)(int64_t m, int64_t n, const double* q, double* out) {
    CP(cplx)* cols = (CP(cplx)*)malloc(sizeof(CP(cplx)) * (size_t)(m * n));
    CP(cplx)* scratch = (CP(cplx)*)malloc(sizeof(CP(cplx)) * (size_t)m);
    CP(load_cols)(cols, q, m, n);
    R worst = CP(rzero)();
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = i; j < n; ++j) {
            CP(cplx) s = CP(tree_inner_product)(cols + i * m, cols + j * m, m, scratch);
            if (i == j) s.re = RP(sub)(s.re, CP(rfrom)(1.0));
            R e = CP(cabs)(s);
            if (RP(lt)(worst, e)) worst = e;
        }
    }
    memcpy(out, &worst, sizeof(R));
    free(cols);
    free(scratch);
}

/* elementwise arithmetic for the parity tests */
static int CP(arith_one)(int op, const double* a, const double* b, double* out) {
    R ra, rb;
    memcpy(&ra, a, sizeof(R));
    memcpy(&rb, b, sizeof(R));
    switch (op) {
        case 0: {
            R o = RP(add)(ra, rb);
            memcpy(out, &o, sizeof(R));
            return 0;
        }
        case 1: {
            R o = RP(sub)(ra, rb);
            memcpy(out, &o, sizeof(R));
            return 0;
        }
        case 2: {
            R o = RP(mul)(ra, rb);
            memcpy(out, &o, sizeof(R));
            return 0;
        }
        case 3: {
            R o = RP(div)(ra, rb);
            memcpy(out, &o, sizeof(R));
            return 0;
        }
        case 4: {
            R o = RP(sqrt)(ra);
            memcpy(out, &o, sizeof(R));
            return 0;
        }
        case 5: CP(store)(out, CP(mul)(CP(load)(a), CP(load)(b))); return 0;
        case 6: CP(store)(out, CP(div)(CP(load)(a), CP(load)(b))); return 0;
        case 7: CP(store)(out, CP(add)(CP(load)(a), CP(load)(b))); return 0;
        default: return XO_USAGE;
    }
}
