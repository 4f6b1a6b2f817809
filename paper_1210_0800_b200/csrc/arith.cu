// arith.cu -- elementwise device arithmetic for the bitwise parity tests
// (per-element semantics in xarith_elem.cuh).
#include "xarith_elem.cuh"
#include "xqr_internal.h"

namespace xb {

template <int L>
__global__ void arith_kernel(int op, int64_t count, const double* a, const double* b, double* out,
                             int32_t* codes) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= count) return;
    const int stride = (op >= 5 && op <= 7) ? 2 * L : L;
    const int code = arith_elem<L>(op, a + e * stride, (b ? b : a) + e * stride, out + e * stride);
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
