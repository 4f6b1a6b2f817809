#pragma once
// Drop-in for xqr/random.hpp (reference random.hpp:17-71): the synthetic
// inputs of every experiment.  SplitMix64 with its published constants and
// the reference's child-stream derivation (a stream is a pure function of
// the parent state and the stream index), and complex samples r*e^{i theta}
// whose modulus spans [10^-g, 10^g] (log-uniform exponent by default, or a
// uniform modulus), computed in double and widened exactly to R.  The C ABI's
// xqr_gen_systems (csrc/gen.cpp) draws the same numbers for whole batches.
#include <cmath>
#include <cstdint>
#include <numbers>

#include "xqr/complex.hpp"
#include "xqr/errors.hpp"

namespace xqr {

class split_mix64 {
public:
    explicit split_mix64(std::uint64_t seed) : state_(seed) {}
    std::uint64_t next() {
        state_ += kGamma;
        return finalize(state_);
    }
    // uniform on [0, 1): the top 53 bits
    double next_unit() { return static_cast<double>(next() >> 11) * 0x1p-53; }
    // child generator for stream k (random.hpp:38-40)
    split_mix64 split(std::uint64_t k) const { return split_mix64(finalize(state_ ^ ((k + 1) * kGamma))); }

private:
    static constexpr std::uint64_t kGamma = 0x9E3779B97F4A7C15ull;
    static std::uint64_t finalize(std::uint64_t z) {
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    std::uint64_t state_;
};

enum class modulus_dist { log_uniform, linear_uniform };

template <class R>
cplx<R> random_unit_complex(split_mix64& rng) {
    const double angle = 2.0 * std::numbers::pi * rng.next_unit();
    return {R(std::cos(angle)), R(std::sin(angle))};
}

// g == 0 is the unit sample (same draws); otherwise the modulus first, then
// the angle (random.hpp:57-71)
template <class R>
cplx<R> random_ranged_complex(split_mix64& rng, double g, modulus_dist dist = modulus_dist::log_uniform) {
    if (g < 0.0) throw usage_error("modulus range exponent must be nonnegative");
    if (g == 0.0) return random_unit_complex<R>(rng);
    double modulus;
    if (dist == modulus_dist::log_uniform) {
        modulus = std::pow(10.0, g * (2.0 * rng.next_unit() - 1.0));
    } else {
        const double lo = std::pow(10.0, -g), hi = std::pow(10.0, g);
        modulus = lo + (hi - lo) * rng.next_unit();
    }
    const double angle = 2.0 * std::numbers::pi * rng.next_unit();
    return {R(modulus * std::cos(angle)), R(modulus * std::sin(angle))};
}

}  // namespace xqr
