// arith_host.cpp -- the product's device arithmetic source
// (paper_1210_0800_b200/csrc/xarith*.cuh) compiled for the host, so the CPU
// test suite can check it bit for bit against the oracle without a GPU.
// Build: g++ -O2 -std=c++17 -ffp-contract=off -shared -fPIC (see tests/test_arith_host.py).
#include <cstdint>

#include "../../paper_1210_0800_b200/csrc/xarith_elem.cuh"

extern "C" int xh_arith(int limbs, int op, int64_t count, const double* a, const double* b,
                        double* out, int32_t* codes) {
    if (limbs != 1 && limbs != 2 && limbs != 4) return 5;
    const int64_t stride = (op >= 5 && op <= 7) ? 2 * limbs : limbs;
    for (int64_t e = 0; e < count; ++e) {
        const double* pa = a + e * stride;
        const double* pb = (b ? b : a) + e * stride;
        double* po = out + e * stride;
        int c = limbs == 1 ? xb::arith_elem<1>(op, pa, pb, po)
                : limbs == 2 ? xb::arith_elem<2>(op, pa, pb, po)
                             : xb::arith_elem<4>(op, pa, pb, po);
        if (codes) codes[e] = c;
    }
    return 0;
}
