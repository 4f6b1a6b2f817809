// test_dropin.cpp -- the reference's own call patterns (test_mgs.cpp,
// test_parallel.cpp) compiled against the drop-in headers in include/xqr/ and
// run on the B200 through libxqr_b200.so; results compared bit for bit with
// the CPU oracle (oracle/xqr_oracle.c, test infrastructure).
// Built by __graft_entry__.build(); run by tests/test_dropin_gpu.py.
#include <cstdio>
#include <cstring>
#include <vector>

#include "xqr/matrix.hpp"
#include "xqr/mgs.hpp"
#include "xqr/parallel.hpp"

extern "C" {
#include "xqr_oracle.h"
}

using namespace xqr;

static int failures = 0, checks = 0;
#define CHECK(c)                                                         \
    do {                                                                 \
        ++checks;                                                        \
        if (!(c)) {                                                      \
            ++failures;                                                  \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
        }                                                                \
    } while (0)

template <class R>
col_matrix<R> from_aos(const std::vector<double>& a, std::size_t m, std::size_t n) {
    col_matrix<R> out(m, n);
    const std::size_t e = 2 * real_traits<R>::components;
    for (std::size_t j = 0; j < n; ++j) std::memcpy(out.column(j).data(), a.data() + j * m * e, m * e * 8);
    return out;
}

template <class R>
bool same_bits(const col_matrix<R>& a, const std::vector<double>& b) {
    const std::size_t e = 2 * real_traits<R>::components;
    for (std::size_t j = 0; j < a.cols(); ++j)
        if (std::memcmp(a.column(j).data(), b.data() + j * a.rows() * e, a.rows() * e * 8)) return false;
    return true;
}

template <class R>
void known_answers() {
    // test_mgs.cpp:45-55 identity factors to identity
    auto f = mgs_qr(col_matrix<R>::identity(4));
    for (std::size_t j = 0; j < 4; ++j)
        for (std::size_t i = 0; i < 4; ++i) {
            cplx<R> expect{R(i == j ? 1.0 : 0.0), R(0.0)};
            CHECK(f.q(i, j) == expect);
            CHECK(f.r(i, j) == expect);
        }
    // test_mgs.cpp:70-90 dependent columns break down at column 2
    col_matrix<R> a(3, 2);
    for (std::size_t i = 0; i < 3; ++i) {
        a(i, 0) = {R(double(i) + 1.0), R(0.5)};
        a(i, 1) = a(i, 0);
    }
    try {
        mgs_qr(a);
        CHECK(false);
    } catch (const breakdown_error& e) {
        CHECK(e.column == 2);
    }
    // test_mgs.cpp:220-228 least squares on the identity returns b, z == 0
    auto eye = col_matrix<R>::identity(3);
    cvector<R> b{{R(1.5), R(-2.0)}, {R(0.25), R(3.0)}, {R(-1.0), R(0.5)}};
    auto sol = lsq_solve(eye, b);
    for (std::size_t i = 0; i < 3; ++i) CHECK(sol.x[i] == b[i]);
    CHECK(sol.residual_norm == R(0.0));
    // mgs.hpp:113-114, :135 dimension errors; :119-121 domain error
    try {
        lsq_solve(eye, cvector<R>(2));
        CHECK(false);
    } catch (const dimension_error&) {
        CHECK(true);
    }
    col_matrix<R> bad(2, 2);
    bad(0, 0) = {R(1.0), R(0.0)};
    try {
        back_substitute(bad, cvector<R>(2));
        CHECK(false);
    } catch (const domain_error&) {
        CHECK(true);
    }
    try {
        worker_pool p(0);
        CHECK(false);
    } catch (const usage_error&) {
        CHECK(true);
    }
}

template <class R>
void random_parity(std::size_t m, std::size_t n, std::uint64_t seed) {
    const int L = (int)real_traits<R>::components;
    const std::size_t e = 2 * L;
    std::vector<double> a(m * n * e), b(m * e);
    xo_gen_system(L, (int64_t)m, (int64_t)n, 1.0, seed, -1, a.data(), b.data());
    std::vector<double> q(a.size()), r(n * n * e), x(n * e), z(L);
    xo_status st{};
    xo_mgs_qr(L, (int64_t)m, (int64_t)n, a.data(), q.data(), r.data(), &st);
    CHECK(st.code == 0);
    auto A = from_aos<R>(a, m, n);
    auto f = mgs_qr(A);
    CHECK(same_bits(f.q, q));
    CHECK(same_bits(f.r, r));
    auto fp = par_mgs_qr(A, 4, normalize_mode::redundant);
    CHECK(same_bits(fp.q, q));
    xo_lsq_solve(L, (int64_t)m, (int64_t)n, a.data(), b.data(), x.data(), z.data(), &st);
    cvector<R> B(m);
    std::memcpy(B.data(), b.data(), b.size() * 8);
    auto sol = par_lsq_solve(A, B, 8);
    CHECK(std::memcmp(sol.x.data(), x.data(), x.size() * 8) == 0);
    CHECK(std::memcmp(&sol.residual_norm, z.data(), z.size() * 8) == 0);
    // verification metrics (mgs.hpp:161-222) on the device == the oracle's
    std::vector<double> res(L), dfc(L);
    xo_residual_max_entry(L, (int64_t)m, (int64_t)n, a.data(), q.data(), r.data(), res.data(), &st);
    xo_orthogonality_defect(L, (int64_t)m, (int64_t)n, q.data(), dfc.data(), &st);
    R gres = residual_max_entry(A, f.q, f.r);
    R gdfc = orthogonality_defect(f.q);
    CHECK(std::memcmp(&gres, res.data(), L * 8) == 0);
    CHECK(std::memcmp(&gdfc, dfc.data(), L * 8) == 0);
    // batched extension
    std::vector<col_matrix<R>> As(3, A);
    std::vector<cvector<R>> Bs(3, B);
    auto br = lsq_solve_batched(As, Bs);
    for (int s = 0; s < 3; ++s) {
        CHECK(br.codes[s] == 0);
        CHECK(std::memcmp(br.solutions[s].x.data(), x.data(), x.size() * 8) == 0);
    }
}

int main() {
    known_answers<double>();
    known_answers<double_double>();
    known_answers<quad_double>();
    random_parity<double>(33, 33, 1);
    random_parity<double_double>(32, 32, 1);
    random_parity<double_double>(45, 20, 9);
    random_parity<quad_double>(24, 24, 3);
    // the single-system grid kernels through the same C++ API: double-double
    // CTA-per-column grid, quad-double clusters (4 CTAs; 8 CTAs with paired
    // bulk updates), and a system taller than one CTA holds (batched: system
    // by system)
    random_parity<double_double>(256, 64, 11);
    random_parity<quad_double>(256, 40, 12);
    random_parity<quad_double>(300, 45, 13);
    random_parity<quad_double>(1100, 5, 14);
    std::printf("%s %d checks, %d failures\n", failures ? "FAIL" : "PASS", checks, failures);
    return failures ? 1 : 0;
}
