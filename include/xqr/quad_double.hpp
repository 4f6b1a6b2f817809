#pragma once
// Drop-in for xqr::quad_double (reference quad_double.hpp:19-385): four limbs
// c[0..3], the same constructors, to_double / to_double_double, the accurate
// add and multiply, division, sqrt, mul_pwr2, renormalize, abs and
// comparisons -- the product's own arithmetic (xarith.cuh built for the
// host), bitwise equal to the reference's, with its exceptions
// (qd_checked :202-205, division :346-355, sqrt :359-370).
#include <array>
#include <cmath>

#include "xqr/detail/host_arith.hpp"
#include "xqr/double_double.hpp"
#include "xqr/errors.hpp"

namespace xqr {

struct quad_double {
    std::array<double, 4> c{0.0, 0.0, 0.0, 0.0};
    constexpr quad_double() = default;
    constexpr quad_double(double d) : c{d, 0.0, 0.0, 0.0} {}
    constexpr quad_double(double c0, double c1, double c2, double c3) : c{c0, c1, c2, c3} {}
    explicit constexpr quad_double(const double_double& d) : c{d.hi, d.lo, 0.0, 0.0} {}
};

inline double to_double(const quad_double& a) { return a.c[0]; }
inline bool isfinite(const quad_double& a) { return std::isfinite(a.c[0]); }

// Round to double-double (quad_double.hpp:30-34): the two leading limbs
// summed exactly, the two trailing ones folded in rounded.
inline double_double to_double_double(const quad_double& a) {
    double s, e, z, ze;
    xb::two_sum(a.c[0], a.c[1], s, e);
    xb::quick_two_sum(s, xb::dadd(e, xb::dadd(a.c[2], a.c[3])), z, ze);
    return {z, ze};
}

namespace detail {
inline xb::r4 xb_of(const quad_double& a) { return {a.c[0], a.c[1], a.c[2], a.c[3]}; }
inline quad_double of_xb(const xb::r4& v) { return {v.c0, v.c1, v.c2, v.c3}; }
inline quad_double qd_checked(const quad_double& a) {
    if (!std::isfinite(a.c[0])) throw overflow_error("quad_double overflow");
    return a;
}
inline quad_double qd_checked(const xb::r4& v) { return qd_checked(of_xb(v)); }
}  // namespace detail

inline quad_double renormalize(const quad_double& a) {
    return detail::of_xb(xb::renormalize(detail::xb_of(a)));
}
inline quad_double operator-(const quad_double& a) { return {-a.c[0], -a.c[1], -a.c[2], -a.c[3]}; }
inline quad_double operator+(const quad_double& a, const quad_double& b) {
    return detail::qd_checked(xb::add(detail::xb_of(a), detail::xb_of(b)));
}
inline quad_double operator-(const quad_double& a, const quad_double& b) { return a + (-b); }
inline quad_double operator*(const quad_double& a, const quad_double& b) {
    return detail::qd_checked(xb::mul(detail::xb_of(a), detail::xb_of(b)));
}
inline quad_double mul_pwr2(const quad_double& a, double p2) {
    return {a.c[0] * p2, a.c[1] * p2, a.c[2] * p2, a.c[3] * p2};
}
inline quad_double operator/(const quad_double& a, const quad_double& b) {
    int status = 0;
    const xb::recip_t<xb::r4> rc = xb::recip(detail::xb_of(b), status);
    if (status == 3) throw domain_error("quad_double division by zero");
    if (status == 2) throw overflow_error("quad_double division overflow");
    return detail::qd_checked(xb::divide(detail::xb_of(a), detail::xb_of(b), rc));
}
inline quad_double sqrt(const quad_double& a) {
    if (a.c[0] == 0.0 && a.c[1] == 0.0 && a.c[2] == 0.0 && a.c[3] == 0.0) return {};
    if (a.c[0] < 0.0) throw domain_error("quad_double sqrt of negative value");
    return detail::qd_checked(xb::rsqrt_ref(detail::xb_of(a)));
}
inline quad_double& operator+=(quad_double& a, const quad_double& b) { return a = a + b; }
inline quad_double& operator-=(quad_double& a, const quad_double& b) { return a = a - b; }
inline quad_double& operator*=(quad_double& a, const quad_double& b) { return a = a * b; }
inline quad_double& operator/=(quad_double& a, const quad_double& b) { return a = a / b; }

inline bool operator==(const quad_double& a, const quad_double& b) { return a.c == b.c; }
inline bool operator!=(const quad_double& a, const quad_double& b) { return !(a == b); }
inline bool operator<(const quad_double& a, const quad_double& b) {
    for (int i = 0; i < 4; ++i) {
        if (a.c[i] < b.c[i]) return true;
        if (a.c[i] > b.c[i]) return false;
    }
    return false;
}
inline bool operator>(const quad_double& a, const quad_double& b) { return b < a; }
inline bool operator<=(const quad_double& a, const quad_double& b) { return !(b < a); }
inline bool operator>=(const quad_double& a, const quad_double& b) { return !(a < b); }

inline quad_double abs(const quad_double& a) { return a.c[0] < 0.0 ? -a : a; }

}  // namespace xqr
