// host_ops.cpp -- the drop-in headers' HOST operators (include/xqr/*.hpp:
// double_double, quad_double, cplx, sqrt, renormalize, and the detail:: MGS
// building blocks of mgs.hpp), exported with the oracle's calling convention
// so the CPU suite can compare them bit for bit (and exception for
// exception) with the reference compiled in place (tests/test_dropin_host.py).
// Build: g++ -std=c++20 -O2 -ffp-contract=off -shared -fPIC -I include.
#include <cstdint>
#include <cstring>
#include <vector>

#include "xqr/mgs.hpp"

using namespace xqr;

namespace {

template <class R>
constexpr int limbs_of() {
    return static_cast<int>(real_traits<R>::components);
}
template <class R>
R ld(const double* p) {
    R v;
    std::memcpy(&v, p, sizeof(R));
    return v;
}
template <class R>
void st(double* p, const R& v) {
    std::memcpy(p, &v, sizeof(R));
}
template <class R>
cplx<R> ldc(const double* p) {
    return {ld<R>(p), ld<R>(p + limbs_of<R>())};
}
template <class R>
void stc(double* p, const cplx<R>& z) {
    st(p, z.re);
    st(p + limbs_of<R>(), z.im);
}

template <class F>
int code_of(F&& f) {
    try {
        f();
    } catch (const breakdown_error&) {
        return 1;
    } catch (const overflow_error&) {
        return 2;
    } catch (const domain_error&) {
        return 3;
    } catch (const dimension_error&) {
        return 4;
    } catch (const usage_error&) {
        return 5;
    }
    return 0;
}

template <class R>
int one(int op, const double* pa, const double* pb, double* po) {
    return code_of([&] {
        switch (op) {
            case 0: st(po, ld<R>(pa) + ld<R>(pb)); break;
            case 1: st(po, ld<R>(pa) - ld<R>(pb)); break;
            case 2: st(po, ld<R>(pa) * ld<R>(pb)); break;
            case 3: st(po, ld<R>(pa) / ld<R>(pb)); break;
            case 4: st(po, xqr::sqrt(ld<R>(pa))); break;
            case 5: stc(po, ldc<R>(pa) * ldc<R>(pb)); break;
            case 6: stc(po, ldc<R>(pa) / ldc<R>(pb)); break;
            case 7: stc(po, ldc<R>(pa) + ldc<R>(pb)); break;
            case 8: st(po, renormalize(ld<R>(pa))); break;
            default: throw usage_error("op");
        }
    });
}

// mgs_qr driven through the detail:: building blocks, the loop of
// test_mgs.cpp:120-146 / acceptance.cpp:497-508
template <class R>
int mgs_by_parts(int64_t m, int64_t n, const double* a, double* q, double* r) {
    constexpr int L = limbs_of<R>();
    return code_of([&] {
        std::vector<cvector<R>> cols(n, cvector<R>(m));
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < m; ++i) cols[j][i] = ldc<R>(a + (j * m + i) * 2 * L);
        cvector<R> scratch(m);
        const R thr = detail::breakdown_threshold<R>((std::size_t)m, detail::max_column_norm(cols, scratch));
        std::vector<cplx<R>> rr(n * n);
        for (int64_t k = 0; k < n; ++k) {
            rr[k * n + k] = cplx<R>{detail::normalize_column(cols[k], scratch, thr, (std::size_t)k + 1), R(0.0)};
            for (int64_t j = k + 1; j < n; ++j) rr[j * n + k] = detail::remove_projection(cols[k], cols[j], scratch);
        }
        for (int64_t j = 0; j < n; ++j) {
            for (int64_t i = 0; i < m; ++i) stc(q + (j * m + i) * 2 * L, cols[j][i]);
            for (int64_t i = 0; i < n; ++i) stc(r + (j * n + i) * 2 * L, rr[j * n + i]);
        }
    });
}

}  // namespace

extern "C" int xq_arith(int limbs, int op, int64_t count, const double* a, const double* b, double* out,
                        int32_t* codes) {
    int bad = 0;
    for (int64_t e = 0; e < count; ++e) {
        const int64_t stride = (op >= 5 && op <= 7) ? 2 * limbs : limbs;
        const double* pa = a + e * stride;
        const double* pb = (b ? b : a) + e * stride;
        double* po = out + e * stride;
        int c = limbs == 1 ? one<double>(op, pa, pb, po)
                : limbs == 2 ? one<double_double>(op, pa, pb, po)
                             : one<quad_double>(op, pa, pb, po);
        if (codes) codes[e] = c;
        bad |= c != 0;
    }
    return bad;
}

extern "C" int xq_mgs_by_parts(int limbs, int64_t m, int64_t n, const double* a, double* q, double* r) {
    switch (limbs) {
        case 1: return mgs_by_parts<double>(m, n, a, q, r);
        case 2: return mgs_by_parts<double_double>(m, n, a, q, r);
        default: return mgs_by_parts<quad_double>(m, n, a, q, r);
    }
}

// real_cast / to_double_double / residual arithmetic spot checks:
// out = [to_double_double(qd) limbs (2), real_cast<qd>(dd) limbs (4), abs2 and cabs of a cqd (8)]
extern "C" void xq_misc(const double* qd4, const double* cqd8, double* out) {
    const quad_double x = ld<quad_double>(qd4);
    st(out, to_double_double(x));
    st(out + 2, real_cast<quad_double>(real_cast<double_double>(x)));
    const cplx<quad_double> z = ldc<quad_double>(cqd8);
    st(out + 6, abs2(z));
    st(out + 10, cabs(z));
}
