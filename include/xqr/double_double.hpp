#pragma once
// Drop-in for xqr::double_double (reference double_double.hpp:15-122): the
// {hi, lo} value type with its constructors, checked arithmetic, sqrt, abs,
// mul_pwr2, renormalize and comparisons.  The arithmetic is the product's own
// (xarith.cuh, built for the host -- detail/host_arith.hpp), bitwise equal to
// the reference's; errors are the reference's exceptions: overflow_error for
// a non-finite leading component (:34-37), domain_error for a zero divisor or
// a negative square root (:81, :96).
#include <cmath>

#include "xqr/detail/host_arith.hpp"
#include "xqr/errors.hpp"

namespace xqr {

struct double_double {
    double hi = 0.0;
    double lo = 0.0;
    constexpr double_double() = default;
    constexpr double_double(double h) : hi(h), lo(0.0) {}
    constexpr double_double(double h, double l) : hi(h), lo(l) {}
};

inline double to_double(const double_double& a) { return a.hi; }
inline bool isfinite(const double_double& a) { return std::isfinite(a.hi); }

namespace detail {
inline xb::r2 xb_of(const double_double& a) { return {a.hi, a.lo}; }
inline double_double of_xb(const xb::r2& v) { return {v.c0, v.c1}; }
inline double_double dd_checked(double hi, double lo) {
    if (!std::isfinite(hi)) throw overflow_error("double_double overflow");
    return {hi, lo};
}
inline double_double dd_checked(const xb::r2& v) { return dd_checked(v.c0, v.c1); }
// double_double.hpp:66-76 (unchecked helpers of the division)
inline double_double dd_add_d(const double_double& a, double b) { return of_xb(xb::dd_add_d(xb_of(a), b)); }
inline double_double dd_mul_d(const double_double& a, double b) { return of_xb(xb::dd_mul_d(xb_of(a), b)); }
}  // namespace detail

inline double_double renormalize(const double_double& a) {
    return detail::of_xb(xb::renormalize(detail::xb_of(a)));
}
inline double_double operator-(const double_double& a) { return {-a.hi, -a.lo}; }
inline double_double operator+(const double_double& a, const double_double& b) {
    return detail::dd_checked(xb::add(detail::xb_of(a), detail::xb_of(b)));
}
inline double_double operator-(const double_double& a, const double_double& b) { return a + (-b); }
inline double_double operator*(const double_double& a, const double_double& b) {
    return detail::dd_checked(xb::mul(detail::xb_of(a), detail::xb_of(b)));
}
inline double_double operator/(const double_double& a, const double_double& b) {
    int status = 0;
    const xb::recip_t<xb::r2> rc = xb::recip(detail::xb_of(b), status);
    if (status == 3) throw domain_error("double_double division by zero");
    if (status == 2) throw overflow_error("double_double division overflow");
    return detail::dd_checked(xb::divide(detail::xb_of(a), detail::xb_of(b), rc));
}
inline double_double sqrt(const double_double& a) {
    if (a.hi == 0.0 && a.lo == 0.0) return {};
    if (a.hi < 0.0) throw domain_error("double_double sqrt of negative value");
    return detail::dd_checked(xb::rsqrt_ref(detail::xb_of(a)));
}
inline double_double& operator+=(double_double& a, const double_double& b) { return a = a + b; }
inline double_double& operator-=(double_double& a, const double_double& b) { return a = a - b; }
inline double_double& operator*=(double_double& a, const double_double& b) { return a = a * b; }
inline double_double& operator/=(double_double& a, const double_double& b) { return a = a / b; }

inline bool operator==(const double_double& a, const double_double& b) {
    return a.hi == b.hi && a.lo == b.lo;
}
inline bool operator!=(const double_double& a, const double_double& b) { return !(a == b); }
inline bool operator<(const double_double& a, const double_double& b) {
    return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo);
}
inline bool operator>(const double_double& a, const double_double& b) { return b < a; }
inline bool operator<=(const double_double& a, const double_double& b) { return !(b < a); }
inline bool operator>=(const double_double& a, const double_double& b) { return !(a < b); }

inline double_double abs(const double_double& a) { return a.hi < 0.0 ? -a : a; }
// exact scaling by a power of two (double_double.hpp:119-122)
inline double_double mul_pwr2(const double_double& a, double p2) { return {a.hi * p2, a.lo * p2}; }

}  // namespace xqr
