// ref_shim.cpp -- CPU ORACLE / reference baseline (test + bench infrastructure only).
//
// Compiles the UNMODIFIED reference headers in place
// (-I/root/reference/proj/include, see oracle/Makefile) and exposes the hot
// path through the same extern "C" signatures as oracle/xqr_oracle.h with a
// `ref_` prefix, plus the reference's own CPU parallel driver (par_lsq_solve,
// parallel.hpp:105-153) and a thread-per-share batch runner used as the CPU
// baseline in bench.py.  Nothing here is product code; the built library
// lives in oracle/_ref/ (git-ignored, not gpurun-ignored).
#include <cstdint>
#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "xqr/experiment.hpp"
#include "xqr/mgs.hpp"
#include "xqr/parallel.hpp"
#include "xqr/random.hpp"
#include "xqr_oracle.h"

using namespace xqr;

namespace {

template <class R>
constexpr int limbs_of() {
    if constexpr (std::is_same_v<R, double>) return 1;
    else if constexpr (std::is_same_v<R, double_double>) return 2;
    else return 4;
}

template <class R>
void load_real(const double* p, R& v) {
    std::memcpy(&v, p, sizeof(R));
}
template <class R>
void store_real(double* p, const R& v) {
    std::memcpy(p, &v, sizeof(R));
}
template <class R>
cplx<R> load_c(const double* p) {
    constexpr int L = limbs_of<R>();
    cplx<R> z;
    load_real(p, z.re);
    load_real(p + L, z.im);
    return z;
}
template <class R>
void store_c(double* p, const cplx<R>& z) {
    constexpr int L = limbs_of<R>();
    store_real(p, z.re);
    store_real(p + L, z.im);
}
template <class R>
col_matrix<R> load_mat(const double* a, int64_t m, int64_t n) {
    constexpr int L = limbs_of<R>();
    col_matrix<R> out(m, n);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) out(i, j) = load_c<R>(a + (j * m + i) * 2 * L);
    return out;
}
template <class R>
void store_mat(double* p, const col_matrix<R>& a) {
    constexpr int L = limbs_of<R>();
    const int64_t m = a.rows(), n = a.cols();
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) store_c(p + (j * m + i) * 2 * L, a(i, j));
}
template <class R>
cvector<R> load_vec(const double* p, int64_t len) {
    constexpr int L = limbs_of<R>();
    cvector<R> v(len);
    for (int64_t i = 0; i < len; ++i) v[i] = load_c<R>(p + i * 2 * L);
    return v;
}
template <class R>
void store_vec(double* p, const cvector<R>& v) {
    constexpr int L = limbs_of<R>();
    for (size_t i = 0; i < v.size(); ++i) store_c(p + i * 2 * L, v[i]);
}

template <class F>
int guarded(xo_status* st, F&& f) {
    int code = 0, column = 0;
    try {
        f();
    } catch (const breakdown_error& e) {
        code = XO_BREAKDOWN;
        column = (int)e.column;
    } catch (const overflow_error&) {
        code = XO_OVERFLOW;
    } catch (const domain_error&) {
        code = XO_DOMAIN;
    } catch (const dimension_error&) {
        code = XO_DIMENSION;
    } catch (const usage_error&) {
        code = XO_USAGE;
    }
    if (st) {
        st->code = code;
        st->column = column;
        st->system = 0;
    }
    return code;
}

template <class Fn>
int by_limbs(int limbs, xo_status* st, Fn&& fn) {
    switch (limbs) {
        case 1: return guarded(st, [&] { fn(double{}); });
        case 2: return guarded(st, [&] { fn(double_double{}); });
        case 4: return guarded(st, [&] { fn(quad_double{}); });
        default:
            if (st) *st = {XO_USAGE, 0, 0};
            return XO_USAGE;
    }
}

}  // namespace

extern "C" {

int ref_mgs_qr(int limbs, int64_t m, int64_t n, const double* a, double* q, double* r,
               xo_status* st) {
    return by_limbs(limbs, st, [&](auto tag) {
        using R = decltype(tag);
        auto f = mgs_qr(load_mat<R>(a, m, n));
        store_mat(q, f.q);
        store_mat(r, f.r);
    });
}

int ref_par_mgs_qr(int limbs, int64_t m, int64_t n, const double* a, double* q, double* r,
                   int workers, int redundant, xo_status* st) {
    return by_limbs(limbs, st, [&](auto tag) {
        using R = decltype(tag);
        auto f = par_mgs_qr(load_mat<R>(a, m, n), (std::size_t)workers,
                            redundant ? normalize_mode::redundant : normalize_mode::designated);
        store_mat(q, f.q);
        store_mat(r, f.r);
    });
}

int ref_lsq_solve(int limbs, int64_t m, int64_t n, const double* a, const double* b, double* x,
                  double* z, xo_status* st) {
    return by_limbs(limbs, st, [&](auto tag) {
        using R = decltype(tag);
        auto sol = lsq_solve(load_mat<R>(a, m, n), load_vec<R>(b, m));
        store_vec(x, sol.x);
        store_real(z, sol.residual_norm);
    });
}

int ref_par_lsq_solve(int limbs, int64_t m, int64_t n, const double* a, const double* b, double* x,
                      double* z, int workers, xo_status* st) {
    return by_limbs(limbs, st, [&](auto tag) {
        using R = decltype(tag);
        auto sol = par_lsq_solve(load_mat<R>(a, m, n), load_vec<R>(b, m), (std::size_t)workers);
        store_vec(x, sol.x);
        store_real(z, sol.residual_norm);
    });
}

int ref_back_substitute(int limbs, int64_t rn, int64_t rc, const double* r, int64_t ylen,
                        const double* y, double* x, xo_status* st) {
    return by_limbs(limbs, st, [&](auto tag) {
        using R = decltype(tag);
        auto xs = back_substitute(load_mat<R>(r, rn, rc), load_vec<R>(y, ylen));
        store_vec(x, xs);
    });
}

int ref_residual_max_entry(int limbs, int64_t m, int64_t n, const double* a, const double* q,
                           const double* r, double* out, xo_status* st) {
    return by_limbs(limbs, st, [&](auto tag) {
        using R = decltype(tag);
        R e = residual_max_entry(load_mat<R>(a, m, n), load_mat<R>(q, m, n), load_mat<R>(r, n, n));
        store_real(out, e);
    });
}

int ref_orthogonality_defect(int limbs, int64_t m, int64_t n, const double* q, double* out,
                             xo_status* st) {
    return by_limbs(limbs, st, [&](auto tag) {
        using R = decltype(tag);
        store_real(out, orthogonality_defect(load_mat<R>(q, m, n)));
    });
}

int ref_gen_system(int limbs, int64_t m, int64_t n, double g, uint64_t seed, int64_t stream,
                   double* a, double* b) {
    return by_limbs(limbs, nullptr, [&](auto tag) {
        using R = decltype(tag);
        split_mix64 root(seed);
        split_mix64 rng = stream >= 0 ? root.split((uint64_t)stream) : root;
        auto am = gen_matrix<R>(rng, m, n, g);
        store_mat(a, am);
        if (b) store_vec(b, gen_rhs<R>(rng, m, g));
    });
}

void ref_splitmix_next(uint64_t seed, int64_t stream, int64_t count, uint64_t* out) {
    split_mix64 root(seed);
    split_mix64 rng = stream >= 0 ? root.split((uint64_t)stream) : root;
    for (int64_t i = 0; i < count; ++i) out[i] = rng.next();
}

int ref_arith(int limbs, int op, int64_t count, const double* a, const double* b, double* out,
              int32_t* st_codes) {
    int bad = 0;
    for (int64_t e = 0; e < count; ++e) {
        int rc = by_limbs(limbs, nullptr, [&](auto tag) {
            using R = decltype(tag);
            constexpr int L = limbs_of<R>();
            const int stride = (op >= 5 && op <= 7) ? 2 * L : L;
            const double* pa = a + e * stride;
            const double* pb = (b ? b : a) + e * stride;
            double* po = out + e * stride;
            R ra, rb;
            load_real(pa, ra);
            load_real(pb, rb);
            switch (op) {
                case 0: store_real(po, R(ra + rb)); break;
                case 1: store_real(po, R(ra - rb)); break;
                case 2: store_real(po, R(ra * rb)); break;
                case 3: store_real(po, R(ra / rb)); break;
                case 4: store_real(po, R(xqr::sqrt(ra))); break;
                case 5: store_c(po, load_c<R>(pa) * load_c<R>(pb)); break;
                case 6: store_c(po, load_c<R>(pa) / load_c<R>(pb)); break;
                case 7: store_c(po, load_c<R>(pa) + load_c<R>(pb)); break;
                case 8: store_real(po, R(xqr::renormalize(ra))); break;
                default: throw usage_error("op");
            }
        });
        if (st_codes) st_codes[e] = rc;
        if (rc) bad = 1;
    }
    return bad;
}

// CPU baseline for the batched workload: `threads` std::threads, each running
// the sequential reference lsq_solve over a contiguous share of systems (the
// reference has no batch API; experiment.hpp:127-137 loops trials serially).
int ref_lsq_solve_batch(int limbs, int64_t batch, int64_t m, int64_t n, const double* a,
                        const double* b, double* x, double* z, int threads, int32_t* codes) {
    if (threads < 1) threads = 1;
    const int L = limbs;
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([=] {
            int64_t lo = batch * t / threads, hi = batch * (t + 1) / threads;
            for (int64_t s = lo; s < hi; ++s) {
                xo_status st{};
                ref_lsq_solve(limbs, m, n, a + s * m * n * 2 * L, b + s * m * 2 * L,
                              x + s * n * 2 * L, z + s * L, &st);
                if (codes) codes[s] = st.code;
            }
        });
    }
    for (auto& th : pool) th.join();
    return 0;
}

// The reference's own accuracy sweep and CSV (run_accuracy_sweep,
// experiment.hpp:157-176; accuracy_csv, :412-433), for the CLI parity test.
// Writes at most `cap` bytes (NUL-terminated) into out; returns the code of
// an exception that escaped the sweep (0 = ok).
int ref_accuracy_csv(int limbs, int64_t m, int64_t n, const double* g, int ng, int64_t trials,
                     uint64_t seed, int linear, char* out, int64_t cap) {
    accuracy_config cfg;
    cfg.precision = limbs == 1 ? precision_tag::d : (limbs == 2 ? precision_tag::dd : precision_tag::qd);
    cfg.m = (std::size_t)m;
    cfg.n = (std::size_t)n;
    cfg.g_values.assign(g, g + ng);
    cfg.trials = (std::size_t)trials;
    cfg.seed = seed;
    cfg.dist = linear ? modulus_dist::linear_uniform : modulus_dist::log_uniform;
    std::string text;
    xo_status st{};
    int rc = guarded(&st, [&] { text = accuracy_csv(run_accuracy_sweep(cfg)); });
    if (cap > 0) {
        const size_t k = std::min(text.size(), (size_t)(cap - 1));
        std::memcpy(out, text.data(), k);
        out[k] = 0;
    }
    return rc;
}

}  // extern "C"
