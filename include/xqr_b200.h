/*
 * xqr_b200.h -- C ABI of the B200-native complex dd/qd MGS least-squares path.
 *
 * Drop-in boundary for the reference `xqr` hot path.  The reference exposes a
 * C++ template API only (no C ABI); each entry point below is
 * what that API's functions bind to, and include/xqr/mgs.hpp +
 * include/xqr/parallel.hpp re-export them under the reference's own names:
 *
 *   xqr_mgs_qr          <- xqr::mgs_qr<R>(col_matrix<R>)          mgs.hpp:84-106
 *   xqr_lsq_solve       <- xqr::lsq_solve<R>(A, b)                 mgs.hpp:131-158
 *   xqr_back_substitute <- xqr::back_substitute<R>(R, y)           mgs.hpp:110-126
 *   (par_mgs_qr / par_lsq_solve / par_back_substitute, parallel.hpp:35-183,
 *    bind to the same three; the device decomposition replaces the worker pool)
 *   xqr_*_batched       <- the reference's serial trial loop
 *                          (experiment.hpp:127-137) as one device launch.
 *
 * Scalars: `limbs` L = 1 (double), 2 (double_double), 4 (quad_double).
 * Memory image ("AoS", identical to the reference's cvector<cplx<R>> storage,
 * complex.hpp:12-19, matrix.hpp:41): column-major; complex entry (i, j) of an
 * m x n matrix starts at double offset ((j*m + i) * 2) * L; the L limbs of the
 * real part come first, then the L limbs of the imaginary part.  Vectors are
 * m x 1 matrices.  A real scalar (z) is L doubles.  Batched arrays put system
 * s at offset s * (one system's size).
 *
 * Errors: the reference throws (errors.hpp:13-51); here every call returns an
 * xqr_code and fills an xqr_status with the first error in the reference's
 * program order.  include/xqr/errors.hpp maps them back to the same exception
 * types (breakdown_error keeps the 1-based column).
 *
 * Threading: an xqr_ctx is single-threaded (one stream, one workspace).  Use
 * one ctx per host thread / device.  Host-pointer calls are synchronous;
 * *_device calls are asynchronous on the ctx stream.
 */
#ifndef XQR_B200_H
#define XQR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    XQR_OK = 0,
    XQR_BREAKDOWN = 1, /* breakdown_error{column} (mgs.hpp:50)               */
    XQR_OVERFLOW = 2,  /* overflow_error (double_double.hpp:34-37, ...)      */
    XQR_DOMAIN = 3,    /* domain_error (mgs.hpp:119-121, complex.hpp:49,63)  */
    XQR_DIMENSION = 4, /* dimension_error (matrix.hpp:16, mgs.hpp:113-114,135) */
    XQR_USAGE = 5,     /* usage_error (bad limbs / unsupported size)         */
    XQR_CUDA = 16      /* CUDA runtime failure (no reference counterpart)     */
} xqr_code;

typedef struct {
    int32_t code;   /* xqr_code                                   */
    int32_t column; /* 1-based column for XQR_BREAKDOWN, else 0    */
    int64_t system; /* index of the failing system (batched calls) */
} xqr_status;

typedef struct xqr_ctx xqr_ctx;

/* Version of this ABI (major*10000 + minor*100 + patch). */
int xqr_version(void);

/* Context: binds a CUDA device, owns a stream and a growable workspace. */
int xqr_ctx_create(int device, xqr_ctx** out);
void xqr_ctx_destroy(xqr_ctx* ctx);
/* Use an external cudaStream_t (NULL = the ctx's own stream). */
int xqr_ctx_set_stream(xqr_ctx* ctx, void* cuda_stream);
void* xqr_ctx_stream(xqr_ctx* ctx);
int xqr_ctx_synchronize(xqr_ctx* ctx);
/* Human-readable text of the last error seen by this ctx. */
const char* xqr_ctx_last_error(xqr_ctx* ctx);

/* ---- host-buffer entry points (synchronous) ---------------------------- */
/* mgs.hpp:84-106: A (m x n) -> Q (m x n), R (n x n, lower triangle +0). */
int xqr_mgs_qr(xqr_ctx* ctx, int limbs, int64_t m, int64_t n, const double* a, double* q,
               double* r, xqr_status* st);
/* mgs.hpp:131-158: A (m x n), b (m) -> x (n), z = residual norm (L doubles). */
int xqr_lsq_solve(xqr_ctx* ctx, int limbs, int64_t m, int64_t n, const double* a,
                  const double* b, double* x, double* z, xqr_status* st);
/* mgs.hpp:110-126: R (rows x cols), y (ylen) -> x (ylen).
 * dimension_error unless rows == cols == ylen. */
int xqr_back_substitute(xqr_ctx* ctx, int limbs, int64_t rows, int64_t cols, const double* r,
                        int64_t ylen, const double* y, double* x, xqr_status* st);

/* Batched: `batch` independent systems of one shape.  st[s] per system; the
 * return value is the first non-zero code (or 0). */
int xqr_mgs_qr_batched(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                       const double* a, double* q, double* r, xqr_status* st);
int xqr_lsq_solve_batched(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                          const double* a, const double* b, double* x, double* z,
                          xqr_status* st);

/* ---- device-buffer entry points (asynchronous on the ctx stream) ------- */
/* Same layouts, device pointers; st is a device array of `batch` statuses.
 * The Jacobian never has to leave the device. */
int xqr_mgs_qr_batched_device(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                              const double* d_a, double* d_q, double* d_r, xqr_status* d_st);
int xqr_lsq_solve_batched_device(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                                 const double* d_a, const double* d_b, double* d_x, double* d_z,
                                 xqr_status* d_st);
int xqr_back_substitute_batched_device(xqr_ctx* ctx, int limbs, int64_t batch, int64_t n,
                                       const double* d_r, const double* d_y, double* d_x,
                                       xqr_status* d_st);

/* ---- verification metrics ------------------------------ */
/* mgs.hpp:161-178: out (L doubles) = max_ij |a_ij - sum_{l<=j} q_il r_lj|
 * (working precision, left-to-right sums); mgs.hpp:208-222: out = max over
 * i <= j of |q_i^H q_j - delta_ij| on the fixed tree.  XQR_OVERFLOW if a
 * value is not finite.  Batched forms: out has batch*L doubles. */
int xqr_residual_max_entry(xqr_ctx* ctx, int limbs, int64_t m, int64_t n, const double* a,
                           const double* q, const double* r, double* out, xqr_status* st);
int xqr_orthogonality_defect(xqr_ctx* ctx, int limbs, int64_t m, int64_t n, const double* q,
                             double* out, xqr_status* st);
int xqr_residual_max_entry_batched(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                                   const double* a, const double* q, const double* r, double* out,
                                   xqr_status* st);
int xqr_orthogonality_defect_batched(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                                     const double* q, double* out, xqr_status* st);
int xqr_residual_max_entry_batched_device(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                                          const double* d_a, const double* d_q, const double* d_r,
                                          double* d_out, xqr_status* d_st);
int xqr_orthogonality_defect_batched_device(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                                            const double* d_q, double* d_out, xqr_status* d_st);

/* ---- synthetic inputs (host) --------------------------------------------- */
/* The reference generator: split_mix64 (random.hpp:17-41), log-uniform
 * modulus in [10^-g, 10^g] computed in double and widened exactly
 * (random.hpp:46-71), A column-major then b (experiment.hpp:64-79).
 * first_stream < 0: one system from split_mix64(seed) itself (batch must be
 * 1); else system s draws from split_mix64(seed).split(first_stream + s).
 * b may be NULL.  Bitwise identical to the reference's draws. */
int xqr_gen_systems(int limbs, int64_t batch, int64_t m, int64_t n, double g, uint64_t seed,
                    int64_t first_stream, int threads, double* a, double* b);
/* Same, with the modulus distribution of random.hpp:44-71 (`--modulus-dist`,
 * xqr_main.cpp:209-213): dist 0 = log_uniform (the default above), 1 =
 * linear_uniform (modulus uniform on [10^-g, 10^g]). */
int xqr_gen_systems_dist(int limbs, int64_t batch, int64_t m, int64_t n, double g, int dist,
                         uint64_t seed, int64_t first_stream, int threads, double* a, double* b);

/* ---- test / instrumentation --------------------------------------------- */
/* Elementwise device arithmetic, op codes as oracle/xqr_oracle.h xo_arith:
 * 0 add, 1 sub, 2 mul, 3 div, 4 sqrt, 5 cmul, 6 cdiv (Smith), 7 cadd,
 * 8 renormalize.  Host buffers; per-element status in codes (may be NULL). */
int xqr_arith(xqr_ctx* ctx, int limbs, int op, int64_t count, const double* a, const double* b,
              double* out, int32_t* codes);
/* Number of kernel launches this ctx has issued (for the bench's
 * gpu_launches claim). */
int64_t xqr_ctx_launch_count(xqr_ctx* ctx);
/* Number of single-system solves this ctx re-routed from the persistent grid
 * kernels to the one-CTA kernel because the grid could not be made
 * co-resident (same results bit for bit; m <= 1024 only). */
int64_t xqr_ctx_grid_fallbacks(xqr_ctx* ctx);
/* FP64 roofline denominator measured on this ctx's device: lane
 * instructions per second of independent DADD (op 0) or DFMA (op 1) chains
 * over every SM (best of three launches). */
int xqr_fp64_peak(xqr_ctx* ctx, int op, double* lane_instr_per_s);
/* Accumulated device time (ms) of the most recent solver launch, measured
 * with CUDA events on the ctx stream (0 if not yet available). */
float xqr_ctx_last_kernel_ms(xqr_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
