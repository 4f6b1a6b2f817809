// xarith_elem.cuh -- one elementwise arithmetic operation with the reference's
// error semantics, shared by the device parity kernel (arith.cu) and the host
// build of the same source (tests/cpp/arith_host.cpp).
//   dd/qd results with a non-finite head -> overflow (double_double.hpp:34-37,
//   quad_double.hpp:202-205); zero divisor -> domain (double_double.hpp:81,
//   quad_double.hpp:347, complex.hpp:49); sqrt of a negative -> domain
//   (double_double.hpp:96, quad_double.hpp:361).  Plain double (L = 1) is
//   unchecked, like the reference's double overloads (real_type.hpp:16-20).
// Op codes: 0 add, 1 sub, 2 mul, 3 div, 4 sqrt, 5 cmul, 6 cdiv (Smith),
// 7 cadd, 8 renormalize.
#pragma once
#include "xarith.cuh"

namespace xb {

template <int L>
XB_DEV int arith_elem(int op, const double* pa, const double* pb, double* po) {
    using R = real_t<L>;
    using C = cx<R>;
    int code = 0;
    if (!(op >= 5 && op <= 7)) {
        R x, y, o;
        load_real<L>(pa, 1, x);
        load_real<L>(pb, 1, y);
        switch (op) {
            case 0: o = add(x, y); break;
            case 1: o = sub(x, y); break;
            case 2: o = mul(x, y); break;
            case 3:
                if constexpr (L == 1)
                    o = div_plain(x, y);
                else
                    o = rdiv(x, y, code);
                break;
            case 4:
                if (L > 1 && !is_zero(x) && head(x) < 0.0) {
                    code = 3;
                    o = x;
                } else {
                    o = rsqrt_ref(x);
                }
                break;
            case 8: o = renormalize(x); break;
            default: code = 5; o = x;
        }
        if (L > 1 && !code && op != 8 && !vfinite(o)) code = 2;
        store_real<L>(po, 1, o);
    } else {
        C x, y, o;
        load_real<L>(pa, 1, x.re);
        load_real<L>(pa + L, 1, x.im);
        load_real<L>(pb, 1, y.re);
        load_real<L>(pb + L, 1, y.im);
        switch (op) {
            case 5: o = cmul(x, y); break;
            case 6: o = cdiv(x, y, code); break;
            default: o = cadd(x, y); break;
        }
        if (L > 1 && !code && !cfinite(o)) code = 2;
        store_real<L>(po, 1, o.re);
        store_real<L>(po + L, 1, o.im);
    }
    return code;
}

}  // namespace xb
