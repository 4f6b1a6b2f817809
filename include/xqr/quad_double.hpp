#pragma once
// Drop-in for the xqr::quad_double value type (reference quad_double.hpp:19-36,
// :372-385): four limbs c[0..3], same constructors and comparisons.
#include <array>
#include <cmath>

#include "xqr/double_double.hpp"

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
inline quad_double operator-(const quad_double& a) { return {-a.c[0], -a.c[1], -a.c[2], -a.c[3]}; }
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

}  // namespace xqr
