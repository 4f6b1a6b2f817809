// arith.cu -- elementwise device arithmetic for the bitwise parity tests.
// Same op codes and the same error semantics as the reference operators:
//   dd/qd results with a non-finite head -> overflow (double_double.hpp:34-37,
//   quad_double.hpp:202-205); zero divisor -> domain (:81, :347, complex.hpp:49);
//   sqrt of a negative -> domain (:96, :361).  Plain double (L = 1) is unchecked,
//   like the reference's double overloads (real_type.hpp:16-20).
#include "xcolumn.cuh"
#include "xqr_internal.h"

namespace xb {

template <int L>
__global__ void arith_kernel(int op, int64_t count, const double* a, const double* b, double* out,
                             int32_t* codes) {
    using R = real_t<L>;
    using C = cx<R>;
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= count) return;
    const bool cplx = (op >= 5 && op <= 7);
    const int stride = cplx ? 2 * L : L;
    const double* pa = a + e * stride;
    const double* pb = (b ? b : a) + e * stride;
    double* po = out + e * stride;
    int code = 0;
    if (!cplx) {
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
        if (L > 1 && !code && op != 8 && !finite(head(o))) code = 2;
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
    if (codes) codes[e] = code;
}

cudaError_t launch_arith(int limbs, int op, int64_t count, const double* a, const double* b,
                         double* out, int32_t* codes, cudaStream_t s) {
    const unsigned blocks = (unsigned)((count + 127) / 128);
    if (count == 0) return cudaSuccess;
    switch (limbs) {
        case 1: arith_kernel<1><<<blocks, 128, 0, s>>>(op, count, a, b, out, codes); break;
        case 2: arith_kernel<2><<<blocks, 128, 0, s>>>(op, count, a, b, out, codes); break;
        case 4: arith_kernel<4><<<blocks, 128, 0, s>>>(op, count, a, b, out, codes); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace xb
