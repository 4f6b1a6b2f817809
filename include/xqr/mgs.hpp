#pragma once
// Drop-in for xqr/mgs.hpp's hot path (reference mgs.hpp:22-32, :84-158):
// mgs_qr, back_substitute and lsq_solve with the reference's signatures,
// value semantics and exception types -- computed on a B200 through the C ABI
// (include/xqr_b200.h, library libxqr_b200.so).  Results are bitwise equal to
// the reference's.  Link with -lxqr_b200.
//
// Device selection: XQR_DEVICE (default 0).  One C-ABI context per host
// thread and device keeps the functions reentrant, as the reference's are
// (SPEC.md:113).
#include <cstdlib>
#include <cstring>
#include <memory>
#include <type_traits>
#include <utility>
#include <vector>

#include "xqr/complex.hpp"
#include "xqr/errors.hpp"
#include "xqr/matrix.hpp"
#include "xqr/real_type.hpp"
#include "xqr/reduction.hpp"
#include "xqr_b200.h"

namespace xqr {

template <class R>
struct qr_factors {
    col_matrix<R> q;
    col_matrix<R> r;
};

template <class R>
struct lsq_solution {
    cvector<R> x;
    R residual_norm;
};

// The MGS building blocks of the reference (mgs.hpp:36-80), for callers that
// drive their own factorisation loop (test_mgs.cpp:123-145,
// acceptance.cpp:497-508).  They run on the host with the value types'
// operators (the product's arithmetic, bitwise equal to the reference's);
// mgs_qr / lsq_solve / back_substitute below are the B200 path.
namespace detail {

// sqrt of Re(a^H a): the imaginary part of a^H a is zero term by term
template <class R>
R column_norm(const cvector<R>& a, cvector<R>& scratch) {
    return sqrt(tree_inner_product<R>(a, a, scratch).re);
}

// a /= ||a|| in place, returns r_kk; breakdown_error(column_index, 1-based)
// when ||a|| <= threshold
template <class R>
R normalize_column(cvector<R>& a, cvector<R>& scratch, const R& threshold, std::size_t column_index) {
    const R rkk = column_norm(a, scratch);
    if (rkk <= threshold) throw breakdown_error(column_index);
    for (auto& entry : a) entry = div_real(entry, rkk);
    return rkk;
}

// r = q^H a, then a -= r q entry by entry; returns r
template <class R>
cplx<R> remove_projection(const cvector<R>& q, cvector<R>& a, cvector<R>& scratch) {
    const cplx<R> r = tree_inner_product<R>(q, a, scratch);
    for (std::size_t i = 0; i < a.size(); ++i) a[i] = a[i] - r * q[i];
    return r;
}

// rows * epsilon * (largest column norm), in R
template <class R>
R breakdown_threshold(std::size_t rows, const R& max_column_norm) {
    return R(static_cast<double>(rows) * real_traits<R>::epsilon) * max_column_norm;
}

template <class R>
R max_column_norm(const std::vector<cvector<R>>& cols, cvector<R>& scratch) {
    R best(0.0);
    for (const auto& col : cols) {
        const R v = column_norm(col, scratch);
        if (v > best) best = v;
    }
    return best;
}

}  // namespace detail

namespace device {

struct ctx_deleter {
    void operator()(xqr_ctx* c) const { xqr_ctx_destroy(c); }
};

inline int default_device() {
    const char* e = std::getenv("XQR_DEVICE");
    return e ? std::atoi(e) : 0;
}

inline xqr_ctx* context() {
    thread_local std::unique_ptr<xqr_ctx, ctx_deleter> ctx;
    if (!ctx) {
        xqr_ctx* c = nullptr;
        if (xqr_ctx_create(default_device(), &c) != XQR_OK)
            throw device_error("xqr: cannot create a CUDA context (no B200 device?)");
        ctx.reset(c);
    }
    return ctx.get();
}

// Map a C-ABI status to the reference's exception (errors.hpp:13-51).
inline void raise_status(int code, const xqr_status& st) {
    switch (code) {
        case XQR_OK: return;
        case XQR_BREAKDOWN: throw breakdown_error(static_cast<std::size_t>(st.column));
        case XQR_OVERFLOW: throw overflow_error("quad/double-double overflow");
        case XQR_DOMAIN: throw domain_error("division by zero");
        case XQR_DIMENSION: throw dimension_error("dimension mismatch");
        case XQR_USAGE: throw usage_error(xqr_ctx_last_error(context()));
        default: throw device_error(xqr_ctx_last_error(context()));
    }
}

template <class R>
constexpr int limbs() {
    return static_cast<int>(real_traits<R>::components);
}

// col_matrix columns -> one contiguous AoS buffer (cplx<R> is 2L doubles).
template <class R>
std::vector<double> pack(const col_matrix<R>& a) {
    const std::size_t m = a.rows(), n = a.cols(), e = 2 * limbs<R>();
    std::vector<double> out(m * n * e);
    for (std::size_t j = 0; j < n; ++j)
        std::memcpy(out.data() + j * m * e, a.column(j).data(), m * e * sizeof(double));
    return out;
}
template <class R>
void unpack(const double* src, col_matrix<R>& a) {
    const std::size_t m = a.rows(), n = a.cols(), e = 2 * limbs<R>();
    for (std::size_t j = 0; j < n; ++j)
        std::memcpy(a.column(j).data(), src + j * m * e, m * e * sizeof(double));
}

}  // namespace device

// mgs.hpp:84-106
template <class R>
qr_factors<R> mgs_qr(col_matrix<R> a) {
    const std::size_t m = a.rows(), n = a.cols();
    std::vector<double> in = device::pack(a);
    std::vector<double> q(in.size()), r(n * n * 2 * device::limbs<R>());
    xqr_status st{};
    int rc = xqr_mgs_qr(device::context(), device::limbs<R>(), (int64_t)m, (int64_t)n, in.data(),
                        q.data(), r.data(), &st);
    device::raise_status(rc, st);
    col_matrix<R> rr(n, n);
    device::unpack(q.data(), a);
    device::unpack(r.data(), rr);
    return {std::move(a), std::move(rr)};
}

// mgs.hpp:110-126
template <class R>
cvector<R> back_substitute(const col_matrix<R>& r, const cvector<R>& y) {
    const std::size_t n = r.cols();
    if (r.rows() != n) throw dimension_error("triangular factor must be square");
    if (y.size() != n) throw dimension_error("right-hand side length mismatch");
    std::vector<double> rin = device::pack(r);
    cvector<R> x(n);
    xqr_status st{};
    int rc = xqr_back_substitute(device::context(), device::limbs<R>(), (int64_t)r.rows(),
                                 (int64_t)n, rin.data(), (int64_t)y.size(),
                                 reinterpret_cast<const double*>(y.data()),
                                 reinterpret_cast<double*>(x.data()), &st);
    device::raise_status(rc, st);
    return x;
}

// mgs.hpp:131-158
template <class R>
lsq_solution<R> lsq_solve(const col_matrix<R>& a, const cvector<R>& b) {
    const std::size_t m = a.rows(), n = a.cols();
    if (b.size() != m) throw dimension_error("right-hand side length mismatch");
    std::vector<double> in = device::pack(a);
    lsq_solution<R> sol{cvector<R>(n), R(0.0)};
    xqr_status st{};
    int rc = xqr_lsq_solve(device::context(), device::limbs<R>(), (int64_t)m, (int64_t)n, in.data(),
                           reinterpret_cast<const double*>(b.data()),
                           reinterpret_cast<double*>(sol.x.data()),
                           reinterpret_cast<double*>(&sol.residual_norm), &st);
    device::raise_status(rc, st);
    return sol;
}

// Batched extension (no reference counterpart beyond its serial trial loop,
// experiment.hpp:127-137): one launch for many systems of one shape.  Each
// system keeps its own status; `codes[s]` / `columns[s]` follow xqr_status.
template <class R>
struct lsq_batch_result {
    std::vector<lsq_solution<R>> solutions;
    std::vector<int> codes;
    std::vector<int> columns;
};

template <class R>
lsq_batch_result<R> lsq_solve_batched(const std::vector<col_matrix<R>>& a,
                                      const std::vector<cvector<R>>& b) {
    lsq_batch_result<R> out;
    if (a.size() != b.size()) throw dimension_error("batch size mismatch");
    if (a.empty()) return out;
    const std::size_t m = a[0].rows(), n = a[0].cols(), e = 2 * device::limbs<R>();
    std::vector<double> ain(a.size() * m * n * e), bin(a.size() * m * e);
    for (std::size_t s = 0; s < a.size(); ++s) {
        if (a[s].rows() != m || a[s].cols() != n || b[s].size() != m)
            throw dimension_error("batched systems must share one shape");
        std::vector<double> p = device::pack(a[s]);
        std::memcpy(ain.data() + s * m * n * e, p.data(), p.size() * sizeof(double));
        std::memcpy(bin.data() + s * m * e, b[s].data(), m * e * sizeof(double));
    }
    std::vector<double> x(a.size() * n * e), z(a.size() * device::limbs<R>());
    std::vector<xqr_status> st(a.size());
    int rc = xqr_lsq_solve_batched(device::context(), device::limbs<R>(), (int64_t)a.size(),
                                   (int64_t)m, (int64_t)n, ain.data(), bin.data(), x.data(), z.data(),
                                   st.data());
    if (rc >= XQR_DIMENSION) device::raise_status(rc, st[0]);  // shape / usage / device: the whole call
    out.solutions.resize(a.size(), lsq_solution<R>{cvector<R>(n), R(0.0)});
    for (std::size_t s = 0; s < a.size(); ++s) {
        std::memcpy(out.solutions[s].x.data(), x.data() + s * n * e, n * e * sizeof(double));
        std::memcpy(&out.solutions[s].residual_norm, z.data() + s * device::limbs<R>(), sizeof(R));
        out.codes.push_back(st[s].code);
        out.columns.push_back(st[s].column);
    }
    return out;
}

// mgs.hpp:161-178 -- largest entry modulus of A - QR, in working precision.
template <class R>
R residual_max_entry(const col_matrix<R>& a, const col_matrix<R>& q, const col_matrix<R>& r) {
    const std::size_t m = a.rows(), n = a.cols();
    if (q.rows() != m || q.cols() != n || r.rows() != n || r.cols() != n)
        throw dimension_error("factor shapes do not match the input matrix");
    std::vector<double> ai = device::pack(a), qi = device::pack(q), ri = device::pack(r);
    R out{};
    xqr_status st{};
    int rc = xqr_residual_max_entry(device::context(), device::limbs<R>(), (int64_t)m, (int64_t)n,
                                    ai.data(), qi.data(), ri.data(), reinterpret_cast<double*>(&out), &st);
    device::raise_status(rc, st);
    return out;
}

// mgs.hpp:183-204 -- residual_max_entry recomputed with every entry first
// cast to W (real_cast: widening is exact): the same device metric, run in
// W on the cast factors.
template <class W, class R>
W residual_max_entry_widened(const col_matrix<R>& a, const col_matrix<R>& q, const col_matrix<R>& r) {
    const std::size_t m = a.rows(), n = a.cols();
    if (q.rows() != m || q.cols() != n || r.rows() != n || r.cols() != n)
        throw dimension_error("factor shapes do not match the input matrix");
    if constexpr (std::is_same_v<W, R>) {
        return residual_max_entry(a, q, r);
    } else {
        auto cast = [](const col_matrix<R>& x) {
            col_matrix<W> out(x.rows(), x.cols());
            for (std::size_t j = 0; j < x.cols(); ++j)
                for (std::size_t i = 0; i < x.rows(); ++i)
                    out(i, j) = cplx<W>{real_cast<W>(x(i, j).re), real_cast<W>(x(i, j).im)};
            return out;
        };
        return residual_max_entry(cast(a), cast(q), cast(r));
    }
}

// mgs.hpp:208-222 -- largest entry modulus of Q^H Q - I.
template <class R>
R orthogonality_defect(const col_matrix<R>& q) {
    std::vector<double> qi = device::pack(q);
    R out{};
    xqr_status st{};
    int rc = xqr_orthogonality_defect(device::context(), device::limbs<R>(), (int64_t)q.rows(),
                                      (int64_t)q.cols(), qi.data(), reinterpret_cast<double*>(&out), &st);
    device::raise_status(rc, st);
    return out;
}

}  // namespace xqr
