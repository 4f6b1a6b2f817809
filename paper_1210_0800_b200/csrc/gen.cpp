// gen.cpp -- the reference's synthetic-input generator on the host, exported
// through the C ABI so callers (and bench.py) can build the exact systems the
// reference experiments use: split_mix64 (random.hpp:17-41), log-uniform
// ranged complex entries computed in double and widened exactly
// (random.hpp:46-71), A drawn column-major then b (experiment.hpp:64-79).
// Compiled with -ffp-contract=off like the reference; uses the same libm.
#include <cmath>
#include <cstdint>
#include <numbers>
#include <thread>
#include <vector>

#include "../../include/xqr_b200.h"

namespace {

struct split_mix64 {
    uint64_t state;
    static uint64_t mix(uint64_t z) {
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    uint64_t next() {
        state += 0x9E3779B97F4A7C15ull;
        return mix(state);
    }
    double next_unit() { return static_cast<double>(next() >> 11) * 0x1p-53; }
    split_mix64 split(uint64_t k) const { return {mix(state ^ ((k + 1) * 0x9E3779B97F4A7C15ull))}; }
};

// random.hpp:57-71; dist 0 = log_uniform, 1 = linear_uniform
void ranged(split_mix64& rng, double g, int dist, int limbs, double* out) {
    double re, im;
    if (g == 0.0) {
        double theta = 2.0 * std::numbers::pi * rng.next_unit();
        re = std::cos(theta);
        im = std::sin(theta);
    } else {
        double r;
        if (dist == 0) {
            r = std::pow(10.0, g * (2.0 * rng.next_unit() - 1.0));
        } else {
            const double lo = std::pow(10.0, -g);
            const double hi = std::pow(10.0, g);
            r = lo + (hi - lo) * rng.next_unit();
        }
        double theta = 2.0 * std::numbers::pi * rng.next_unit();
        re = r * std::cos(theta);
        im = r * std::sin(theta);
    }
    for (int l = 0; l < 2 * limbs; ++l) out[l] = 0.0;
    out[0] = re;
    out[limbs] = im;
}

void gen_one(int limbs, int64_t m, int64_t n, double g, int dist, split_mix64 rng, double* a, double* b) {
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) ranged(rng, g, dist, limbs, a + (j * m + i) * 2 * limbs);
    if (b)
        for (int64_t i = 0; i < m; ++i) ranged(rng, g, dist, limbs, b + i * 2 * limbs);
}

}  // namespace

extern "C" int xqr_gen_systems_dist(int limbs, int64_t batch, int64_t m, int64_t n, double g,
                                    int dist, uint64_t seed, int64_t first_stream, int threads,
                                    double* a, double* b) {
    if (!(limbs == 1 || limbs == 2 || limbs == 4)) return XQR_USAGE;
    if (dist != 0 && dist != 1) return XQR_USAGE;
    if (g < 0.0) return XQR_USAGE;  // random.hpp:59
    if (n < 1 || m < n) return XQR_DIMENSION;
    if (batch < 0 || (first_stream < 0 && batch > 1)) return XQR_USAGE;
    const split_mix64 root{seed};
    const int64_t asz = m * n * 2 * limbs, bsz = m * 2 * limbs;
    auto work = [&](int64_t lo, int64_t hi) {
        for (int64_t s = lo; s < hi; ++s) {
            split_mix64 rng = first_stream < 0 ? root : root.split((uint64_t)(first_stream + s));
            gen_one(limbs, m, n, g, dist, rng, a + s * asz, b ? b + s * bsz : nullptr);
        }
    };
    if (threads < 1) threads = 1;
    if (threads == 1 || batch < 2) {
        work(0, batch);
        return XQR_OK;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work, batch * t / threads, batch * (t + 1) / threads);
    for (auto& th : pool) th.join();
    return XQR_OK;
}

extern "C" int xqr_gen_systems(int limbs, int64_t batch, int64_t m, int64_t n, double g,
                               uint64_t seed, int64_t first_stream, int threads, double* a,
                               double* b) {
    return xqr_gen_systems_dist(limbs, batch, m, n, g, 0, seed, first_stream, threads, a, b);
}
