#pragma once
// Drop-in for the xqr::double_double value type (reference
// double_double.hpp:15-22, :106-117): same layout {hi, lo}, constructors,
// comparisons and accessors.  Arithmetic on these values happens on the
// B200 inside the solver kernels (paper_1210_0800_b200/csrc/xarith.cuh).
#include <cmath>

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
inline double_double operator-(const double_double& a) { return {-a.hi, -a.lo}; }
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

}  // namespace xqr
