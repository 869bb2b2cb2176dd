// Seeded signal sources of the reference harness, restated so the product's
// benchmark and tests draw exactly the reference's inputs:
//   Rng (mt19937_64 + explicit Box-Muller)  proj/include/dctplus/signal.hpp:18-46
//   gen_ar_signal                          signal.hpp:49-55
//   mix_seed                               bench.hpp:89-95
// plus the 2-D separable AR(1) row source of config 4 (SURVEY.md 8d note),
// which the reference does not have.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <numbers>
#include <random>
#include <stdexcept>
#include <vector>

namespace dctp::host {

class Rng {
  public:
    explicit Rng(std::uint64_t seed) : gen_(seed) {}
    double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
    double gaussian() {
        if (spare_ready_) {
            spare_ready_ = false;
            return spare_;
        }
        double u1;
        do {
            u1 = uniform();
        } while (u1 <= 0.0);
        const double u2 = uniform();
        const double radius = std::sqrt(-2.0 * std::log(u1));
        const double angle = 2.0 * std::numbers::pi * u2;
        spare_ = radius * std::sin(angle);
        spare_ready_ = true;
        return radius * std::cos(angle);
    }

  private:
    std::mt19937_64 gen_;
    bool spare_ready_ = false;
    double spare_ = 0.0;
};

inline std::uint64_t mix_seed(std::uint64_t seed, std::size_t size, std::size_t kind) {
    std::uint64_t x = seed * 0x9e3779b97f4a7c15ULL + size * 0x100000001b3ULL + kind + 1;
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    return x;
}

/// Stationary AR(1): s_0 ~ N(0, 1/(1-r^2)), s_{j+1} = r s_j + N(0, 1).
inline void ar_row(std::size_t n, double r, Rng& rng, double* out) {
    if (!(std::abs(r) < 1.0)) throw std::invalid_argument("gen_ar_signal: need |r| < 1");
    out[0] = rng.gaussian() / std::sqrt(1.0 - r * r);
    for (std::size_t j = 1; j < n; ++j) out[j] = r * out[j - 1] + rng.gaussian();
}

enum class Dist : int { gaussian = 0, uniform = 1, ar = 2, sym_uniform = 3, ar2d = 4 };

/// rows x n samples, row-major, drawn in row order from one Rng(seed).
inline void fill_signals(std::uint64_t seed, Dist dist, double r, std::size_t n, std::size_t rows,
                         double* out) {
    Rng rng(seed);
    switch (dist) {
        case Dist::gaussian:
            for (std::size_t i = 0; i < n * rows; ++i) out[i] = rng.gaussian();
            return;
        case Dist::uniform:
            for (std::size_t i = 0; i < n * rows; ++i) out[i] = rng.uniform();
            return;
        case Dist::sym_uniform:
            for (std::size_t i = 0; i < n * rows; ++i) out[i] = 2.0 * rng.uniform() - 1.0;
            return;
        case Dist::ar:
            for (std::size_t b = 0; b < rows; ++b) ar_row(n, r, rng, out + b * n);
            return;
        case Dist::ar2d: {
            // Fields of n x n: AR(1) rows along the signal axis, then an AR(1)
            // recursion across rows, y_r = r y_{r-1} + sqrt(1-r^2) x_r, so every
            // row is marginally the same stationary AR(1) as gen_ar_signal.
            const double c = std::sqrt(1.0 - r * r);
            std::vector<double> x(n);
            for (std::size_t b = 0; b < rows; ++b) {
                ar_row(n, r, rng, x.data());
                double* y = out + b * n;
                if (b % n == 0) {
                    for (std::size_t j = 0; j < n; ++j) y[j] = x[j];
                } else {
                    const double* prev = y - n;
                    for (std::size_t j = 0; j < n; ++j) y[j] = r * prev[j] + c * x[j];
                }
            }
            return;
        }
    }
    throw std::invalid_argument("fill_signals: unknown distribution");
}

} // namespace dctp::host
