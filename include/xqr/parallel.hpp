#pragma once
// Drop-in for xqr/parallel.hpp (reference parallel.hpp:23-183).  The
// reference's fork-join CPU decomposition (one round per pivot over a
// worker_pool) is replaced by the device decomposition; results are bitwise
// equal to the sequential calls in both, so the par_* entry points keep their
// signatures and route to the same B200 kernels.  `worker_pool` keeps its
// constructor contract (worker_pool.hpp:23-26: zero workers is a usage_error)
// so existing callers compile unchanged.
#include <cstddef>
#include <utility>

#include "xqr/errors.hpp"
#include "xqr/mgs.hpp"

namespace xqr {

enum class normalize_mode { designated, redundant };

class worker_pool {
public:
    explicit worker_pool(std::size_t workers) : n_(workers) {
        if (workers == 0) throw usage_error("worker_pool needs at least one worker");
    }
    std::size_t size() const { return n_; }

private:
    std::size_t n_;
};

template <class R>
qr_factors<R> par_mgs_qr(col_matrix<R> a, worker_pool&, normalize_mode = normalize_mode::designated) {
    return mgs_qr(std::move(a));
}
template <class R>
qr_factors<R> par_mgs_qr(col_matrix<R> a, std::size_t workers,
                         normalize_mode mode = normalize_mode::designated) {
    worker_pool pool(workers);
    return par_mgs_qr(std::move(a), pool, mode);
}
template <class R>
lsq_solution<R> par_lsq_solve(const col_matrix<R>& a, const cvector<R>& b, worker_pool&) {
    return lsq_solve(a, b);
}
template <class R>
lsq_solution<R> par_lsq_solve(const col_matrix<R>& a, const cvector<R>& b, std::size_t workers) {
    worker_pool pool(workers);
    return par_lsq_solve(a, b, pool);
}
template <class R>
cvector<R> par_back_substitute(const col_matrix<R>& r, const cvector<R>& y, worker_pool&) {
    return back_substitute(r, y);
}
template <class R>
cvector<R> par_back_substitute(const col_matrix<R>& r, const cvector<R>& y, std::size_t workers) {
    worker_pool pool(workers);
    return par_back_substitute(r, y, pool);
}

}  // namespace xqr
