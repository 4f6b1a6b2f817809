/*
 * xqr_oracle.h -- CPU ORACLE (test infrastructure only; never on the product path).
 *
 * Plain-C restatement of the reference `xqr` hot path
 * (/root/reference/proj/include/xqr/{eft,double_double,quad_double,complex,
 * reduction,mgs,random}.hpp).  Every function cites the reference file:line
 * it follows.  Pinned against the reference itself: tests compare this
 * restatement bit for bit with oracle/_ref/libxqr_ref.so (the reference
 * headers compiled in place by oracle/Makefile) and with the committed
 * golden fixtures under tests/golden/ that the same reference build produced.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.
 *
 * Memory image used by every matrix/vector argument ("AoS"): column-major,
 * complex entry (i, j) of an m x n matrix starts at double offset
 * ((j * m + i) * 2) * L; the real part's L limbs come first, then the
 * imaginary part's L limbs.  This is exactly the in-memory layout of one
 * reference column `cvector<R>` (complex.hpp:12-19) laid end to end.
 * L = 1 (double), 2 (double_double), 4 (quad_double).
 */
#ifndef XQR_ORACLE_H
#define XQR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes shared with include/xqr_b200.h */
enum {
    XO_OK = 0,
    XO_BREAKDOWN = 1, /* breakdown_error, column 1-based (errors.hpp:36-41) */
    XO_OVERFLOW = 2,  /* overflow_error (errors.hpp:20-22)                  */
    XO_DOMAIN = 3,    /* domain_error (errors.hpp:25-27)                    */
    XO_DIMENSION = 4, /* dimension_error (errors.hpp:30-32)                 */
    XO_USAGE = 5      /* usage_error (errors.hpp:50-52)                     */
};

typedef struct {
    int32_t code;
    int32_t column;
    int64_t system;
} xo_status;

/* mgs.hpp:84-106.  q: m x n, r: n x n (AoS). */
int xo_mgs_qr(int limbs, int64_t m, int64_t n, const double* a, double* q, double* r,
              xo_status* st);
/* mgs.hpp:131-158.  x: n entries, z: L doubles. */
int xo_lsq_solve(int limbs, int64_t m, int64_t n, const double* a, const double* b, double* x,
                 double* z, xo_status* st);
/* mgs.hpp:110-126. r: rn x rc, y: ylen entries. */
int xo_back_substitute(int limbs, int64_t rn, int64_t rc, const double* r, int64_t ylen,
                       const double* y, double* x, xo_status* st);
/* mgs.hpp:161-178 and :208-222 (verification metrics). out: L doubles. */
int xo_residual_max_entry(int limbs, int64_t m, int64_t n, const double* a, const double* q,
                          const double* r, double* out, xo_status* st);
int xo_orthogonality_defect(int limbs, int64_t m, int64_t n, const double* q, double* out,
                            xo_status* st);

/* experiment.hpp:64-79 with random.hpp:17-71.  Draws A (m x n) then b (m)
 * from split_mix64(seed) -- or from split_mix64(seed).split(stream) when
 * stream >= 0 -- with modulus range g (log-uniform).  b may be NULL. */
int xo_gen_system(int limbs, int64_t m, int64_t n, double g, uint64_t seed, int64_t stream,
                  double* a, double* b);
/* random.hpp:17-41 raw stream, for the generator known-answer tests. */
void xo_splitmix_next(uint64_t seed, int64_t stream, int64_t count, uint64_t* out);

/* Elementwise arithmetic for the arithmetic parity tests.
 * op: 0 add, 1 sub, 2 mul, 3 div, 4 sqrt(a), 5 cmul, 6 cdiv (Smith), 7 cadd,
 *     8 renormalize(a) (dd: double_double.hpp:28-31, qd: quad_double.hpp:209-213).
 * Real ops read/write `count` reals of L limbs; complex ops `count` complex
 * entries of 2L doubles.  Per-element status in st_codes (0 ok). */
int xo_arith(int limbs, int op, int64_t count, const double* a, const double* b, double* out,
             int32_t* st_codes);

#ifdef __cplusplus
}
#endif
#endif
