/*
 * xqr_oracle.c -- CPU ORACLE (test infrastructure only; never on the product
 * path).  See xqr_oracle.h for the contract and the pinning story.
 */
#include "xqr_oracle.h"

#include <stdlib.h>
#include <string.h>

#include "xqr_oracle_arith.h"

_Thread_local xo_catch* xo_cur_catch = NULL;

void xo_throw(int code, int column) {
    xo_catch* c = xo_cur_catch;
    if (!c) abort();
    c->code = code;
    c->column = column;
    longjmp(c->env, 1);
}

/* ---- instantiate the algorithm template for d / dd / qd ------------------ */
#define R xo_d
#define RP(x) xo_d_##x
#define CP(x) xd_##x
#define LIMBS 1
#define EPSILON 0x1p-52
#include "xqr_oracle_tmpl.h"
#undef R
#undef RP
#undef CP
#undef LIMBS
#undef EPSILON

#define R xo_dd
#define RP(x) xo_dd_##x
#define CP(x) xdd_##x
#define LIMBS 2
#define EPSILON 0x1p-104
#include "xqr_oracle_tmpl.h"
#undef R
#undef RP
#undef CP
#undef LIMBS
#undef EPSILON

#define R xo_qd
#define RP(x) xo_qd_##x
#define CP(x) xqd_##x
#define LIMBS 4
#define EPSILON 0x1p-209
#include "xqr_oracle_tmpl.h"
#undef R
#undef RP
#undef CP
#undef LIMBS
#undef EPSILON

/* ---- exception boundary --------------------------------------------------- */
#define XO_TRY(st)                           \
    xo_catch catch_;                         \
    xo_catch* saved_ = xo_cur_catch;         \
    xo_cur_catch = &catch_;                  \
    if (setjmp(catch_.env)) {                \
        xo_cur_catch = saved_;               \
        if (st) {                            \
            (st)->code = catch_.code;        \
            (st)->column = catch_.column;    \
            (st)->system = 0;                \
        }                                    \
        return catch_.code;                  \
    }
#define XO_END(st)                        \
    xo_cur_catch = saved_;                \
    if (st) {                             \
        (st)->code = 0;                   \
        (st)->column = 0;                 \
        (st)->system = 0;                 \
    }                                     \
    return 0;

static int xo_fail(xo_status* st, int code) {
    if (st) {
        st->code = code;
        st->column = 0;
        st->system = 0;
    }
    return code;
}

int xo_mgs_qr(int limbs, int64_t m, int64_t n, const double* a, double* q, double* r,
              xo_status* st) {
    /* matrix.hpp:15-19: rows >= cols >= 1 */
    if (n <= 0 || m < n) return xo_fail(st, XO_DIMENSION);
    XO_TRY(st)
    switch (limbs) {
        case 1: xd_mgs_qr(m, n, a, q, r); break;
        case 2: xdd_mgs_qr(m, n, a, q, r); break;
        case 4: xqd_mgs_qr(m, n, a, q, r); break;
        default: xo_throw(XO_USAGE, 0);
    }
    XO_END(st)
}

int xo_lsq_solve(int limbs, int64_t m, int64_t n, const double* a, const double* b, double* x,
                 double* z, xo_status* st) {
    if (n <= 0 || m < n) return xo_fail(st, XO_DIMENSION);
    XO_TRY(st)
    switch (limbs) {
        case 1: xd_lsq_solve(m, n, a, b, x, z); break;
        case 2: xdd_lsq_solve(m, n, a, b, x, z); break;
        case 4: xqd_lsq_solve(m, n, a, b, x, z); break;
        default: xo_throw(XO_USAGE, 0);
    }
    XO_END(st)
}

int xo_back_substitute(int limbs, int64_t rn, int64_t rc, const double* r, int64_t ylen,
                       const double* y, double* x, xo_status* st) {
    /* mgs.hpp:113-114 */
    if (rn != rc) return xo_fail(st, XO_DIMENSION);
    if (ylen != rc) return xo_fail(st, XO_DIMENSION);
    XO_TRY(st)
    switch (limbs) {
        case 1: xd_back_substitute(rc, r, y, x); break;
        case 2: xdd_back_substitute(rc, r, y, x); break;
        case 4: xqd_back_substitute(rc, r, y, x); break;
        default: xo_throw(XO_USAGE, 0);
    }
    XO_END(st)
}

int xo_residual_max_entry(int limbs, int64_t m, int64_t n, const double* a, const double* q,
                          const double* r, double* out, xo_status* st) {
    XO_TRY(st)
    switch (limbs) {
        case 1: xd_residual_max_entry(m, n, a, q, r, out); break;
        case 2: xdd_residual_max_entry(m, n, a, q, r, out); break;
        case 4: xqd_residual_max_entry(m, n, a, q, r, out); break;
        default: xo_throw(XO_USAGE, 0);
    }
    XO_END(st)
}

int xo_orthogonality_defect(int limbs, int64_t m, int64_t n, const double* q, double* out,
                            xo_status* st) {
    XO_TRY(st)
    switch (limbs) {
        case 1: xd_orthogonality_defect(m, n, q, out); break;
        case 2: xdd_orthogonality_defect(m, n, q, out); break;
        case 4: xqd_orthogonality_defect(m, n, q, out); break;
        default: xo_throw(XO_USAGE, 0);
    }
    XO_END(st)
}

/* ---- random.hpp:17-41 ----------------------------------------------------- */
typedef struct {
    uint64_t state;
} xo_rng;

static uint64_t xo_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t xo_next(xo_rng* g) {
    g->state += 0x9E3779B97F4A7C15ull;
    return xo_mix(g->state);
}
static double xo_next_unit(xo_rng* g) { return (double)(xo_next(g) >> 11) * 0x1p-53; }
static xo_rng xo_split(const xo_rng* g, uint64_t k) {
    xo_rng c = {xo_mix(g->state ^ ((k + 1) * 0x9E3779B97F4A7C15ull))};
    return c;
}

static const double xo_pi = 3.141592653589793238462643383279502884; /* std::numbers::pi */

/* random.hpp:46-50 and :56-71 (log-uniform modulus), widened exactly: the
 * real part's limb 0 holds the double, the other limbs are +0. */
static void xo_ranged_complex(xo_rng* g, double gexp, int limbs, double* out) {
    double re, im;
    if (gexp == 0.0) {
        double theta = 2.0 * xo_pi * xo_next_unit(g);
        re = cos(theta);
        im = sin(theta);
    } else {
        double r = pow(10.0, gexp * (2.0 * xo_next_unit(g) - 1.0));
        double theta = 2.0 * xo_pi * xo_next_unit(g);
        re = r * cos(theta);
        im = r * sin(theta);
    }
    for (int l = 0; l < 2 * limbs; ++l) out[l] = 0.0;
    out[0] = re;
    out[limbs] = im;
}

int xo_gen_system(int limbs, int64_t m, int64_t n, double g, uint64_t seed, int64_t stream,
                  double* a, double* b) {
    if (g < 0.0) return XO_USAGE; /* random.hpp:59 */
    xo_rng root = {seed};
    xo_rng rng = stream >= 0 ? xo_split(&root, (uint64_t)stream) : root;
    /* experiment.hpp:64-71: column index outer, row index inner */
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) xo_ranged_complex(&rng, g, limbs, a + (j * m + i) * 2 * limbs);
    /* experiment.hpp:74-79 */
    if (b)
        for (int64_t i = 0; i < m; ++i) xo_ranged_complex(&rng, g, limbs, b + i * 2 * limbs);
    return 0;
}

void xo_splitmix_next(uint64_t seed, int64_t stream, int64_t count, uint64_t* out) {
    xo_rng root = {seed};
    xo_rng rng = stream >= 0 ? xo_split(&root, (uint64_t)stream) : root;
    for (int64_t i = 0; i < count; ++i) out[i] = xo_next(&rng);
}

/* ---- elementwise arithmetic ---------------------------------------------- */
static int xo_arith_one(int limbs, int op, const double* a, const double* b, double* out) {
    xo_catch catch_;
    xo_catch* saved_ = xo_cur_catch;
    xo_cur_catch = &catch_;
    if (setjmp(catch_.env)) {
        xo_cur_catch = saved_;
        return catch_.code;
    }
    int rc;
    if (op == 8) { /* renormalize */
        if (limbs == 2) {
            xo_dd v = xo_dd_renormalize(xo_dd_make(a[0], a[1]));
            out[0] = v.hi;
            out[1] = v.lo;
        } else if (limbs == 4) {
            xo_qd v = xo_qd_renormalize(xo_qd_make(a[0], a[1], a[2], a[3]));
            memcpy(out, v.c, sizeof v.c);
        } else {
            out[0] = a[0];
        }
        rc = 0;
    } else if (limbs == 1) {
        rc = xd_arith_one(op, a, b, out);
    } else if (limbs == 2) {
        rc = xdd_arith_one(op, a, b, out);
    } else if (limbs == 4) {
        rc = xqd_arith_one(op, a, b, out);
    } else {
        rc = XO_USAGE;
    }
    xo_cur_catch = saved_;
    return rc;
}

int xo_arith(int limbs, int op, int64_t count, const double* a, const double* b, double* out,
             int32_t* st_codes) {
    int stride = (op >= 5 && op <= 7) ? 2 * limbs : limbs;
    int bad = 0;
    for (int64_t e = 0; e < count; ++e) {
        int rc = xo_arith_one(limbs, op, a + e * stride, b ? b + e * stride : a + e * stride,
                              out + e * stride);
        if (st_codes) st_codes[e] = rc;
        if (rc) bad = 1;
    }
    return bad ? 1 : 0;
}
