// Host-side real-to-real trigonometric transforms (per-graph setup only).
//
// The reference computes z = dct2(v) and the column signs sigma through
// FFTW r2r plans (proj/include/dctplus/trig.hpp:45-53, :95-114).  FFTW is not
// present in this image, so this header restates the published FFTW kind
// definitions on top of one small complex FFT:
//
//   REDFT10 : Y_k = 2 sum_j x_j cos(pi (2j+1) k / 2n)             (DCT-II)
//   REDFT01 : Y_k = x_0 + 2 sum_{j>=1} x_j cos(pi j (2k+1) / 2n)  (DCT-III)
//   RODFT00 : Y_k = 2 sum_j x_j sin(pi (j+1)(k+1) / (n+1))        (DST-I)
//   DFT     : Y_k = sum_j x_j exp(sign * 2 pi i j k / N)
//
// The per-graph setup (secular roots, normalisers, signs) is bit-sensitive to
// z, so the product's host setup and the FFTW stand-in
// used by the oracle build (oracle/fftw_shim/fftw3.h) execute this one
// implementation: the same inputs give the same bits on both sides.
//
// Everything here is host code compiled with -ffp-contract=off; it is never
// on the batched apply path (the GPU kernels do that).
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <numbers>
#include <stdexcept>
#include <vector>

namespace dctp::r2r {

/// Complex DFT of fixed length and sign on interleaved (re, im) doubles.
/// Radix-2 decimation in time for power-of-two lengths, direct summation with
/// an exact twiddle table otherwise.  Immutable after construction.
class Fft {
  public:
    Fft() = default;
    Fft(std::size_t n, int sign) : n_(n), sign_(sign < 0 ? -1 : 1) {
        if (n == 0) throw std::invalid_argument("r2r::Fft: length must be positive");
        pow2_ = (n & (n - 1)) == 0;
        const double pi = std::numbers::pi;
        const std::size_t nt = pow2_ ? (n / 2 > 0 ? n / 2 : 1) : n;
        w_.resize(2 * nt);
        for (std::size_t k = 0; k < nt; ++k) {
            const double ang = 2.0 * pi * static_cast<double>(k) / static_cast<double>(n);
            w_[2 * k] = std::cos(ang);
            w_[2 * k + 1] = static_cast<double>(sign_) * std::sin(ang);
        }
        if (pow2_) {
            unsigned bits = 0;
            while ((std::size_t{1} << bits) < n) ++bits;
            rev_.resize(n);
            for (std::size_t i = 0; i < n; ++i) {
                std::size_t r = 0;
                for (unsigned b = 0; b < bits; ++b)
                    if (i & (std::size_t{1} << b)) r |= std::size_t{1} << (bits - 1 - b);
                rev_[i] = static_cast<std::uint32_t>(r);
            }
        }
    }

    std::size_t size() const { return n_; }

    /// out = DFT(in); in and out hold 2*size() doubles and must not alias.
    void exec(const double* in, double* out) const {
        const std::size_t n = n_;
        if (!pow2_) {
            for (std::size_t k = 0; k < n; ++k) {
                double ar = 0.0, ai = 0.0;
                std::size_t idx = 0;
                for (std::size_t j = 0; j < n; ++j) {
                    const double wr = w_[2 * idx], wi = w_[2 * idx + 1];
                    const double xr = in[2 * j], xi = in[2 * j + 1];
                    ar += xr * wr - xi * wi;
                    ai += xr * wi + xi * wr;
                    idx += k;
                    if (idx >= n) idx -= n;
                }
                out[2 * k] = ar;
                out[2 * k + 1] = ai;
            }
            return;
        }
        for (std::size_t i = 0; i < n; ++i) {
            out[2 * rev_[i]] = in[2 * i];
            out[2 * rev_[i] + 1] = in[2 * i + 1];
        }
        for (std::size_t len = 2; len <= n; len <<= 1) {
            const std::size_t half = len >> 1, step = n / len;
            for (std::size_t i = 0; i < n; i += len) {
                double* a = out + 2 * i;
                double* b = out + 2 * (i + half);
                for (std::size_t j = 0; j < half; ++j) {
                    const double wr = w_[2 * j * step], wi = w_[2 * j * step + 1];
                    const double br = b[2 * j], bi = b[2 * j + 1];
                    const double tr = br * wr - bi * wi;
                    const double ti = br * wi + bi * wr;
                    const double ar = a[2 * j], ai = a[2 * j + 1];
                    b[2 * j] = ar - tr;
                    b[2 * j + 1] = ai - ti;
                    a[2 * j] = ar + tr;
                    a[2 * j + 1] = ai + ti;
                }
            }
        }
    }

  private:
    std::size_t n_ = 0;
    int sign_ = -1;
    bool pow2_ = true;
    std::vector<double> w_;
    std::vector<std::uint32_t> rev_;
};

enum class Kind { redft10, redft01, rodft00 };

/// One r2r transform of fixed kind and length (FFTW's unnormalised
/// conventions).  exec() needs a scratch of scratch_size() doubles.
class R2r {
  public:
    R2r() = default;
    R2r(Kind kind, std::size_t n) : kind_(kind), n_(n) {
        if (n == 0) throw std::invalid_argument("r2r: length must be positive");
        const double pi = std::numbers::pi;
        switch (kind) {
            case Kind::redft10:
            case Kind::redft01: {
                fft_ = Fft(n, kind == Kind::redft10 ? -1 : +1);
                rot_.resize(2 * n);
                for (std::size_t k = 0; k < n; ++k) {
                    const double ang = pi * static_cast<double>(k) / (2.0 * static_cast<double>(n));
                    rot_[2 * k] = std::cos(ang);
                    rot_[2 * k + 1] = std::sin(ang);
                }
                break;
            }
            case Kind::rodft00:
                fft_ = Fft(2 * (n + 1), -1);
                break;
        }
    }

    Kind kind() const { return kind_; }
    std::size_t size() const { return n_; }
    std::size_t scratch_size() const { return 4 * fft_.size(); }

    void exec(const double* in, double* out, double* scratch) const {
        const std::size_t n = n_;
        double* a = scratch;
        double* b = scratch + 2 * fft_.size();
        switch (kind_) {
            case Kind::redft10: {
                // Makhoul: v = (x0, x2, x4, ..., x5, x3, x1); Y_k = 2 Re(e^{-i pi k/2n} V_k).
                for (std::size_t j = 0; 2 * j < n; ++j) {
                    a[2 * j] = in[2 * j];
                    a[2 * j + 1] = 0.0;
                }
                for (std::size_t j = 0; 2 * j + 1 < n; ++j) {
                    a[2 * (n - 1 - j)] = in[2 * j + 1];
                    a[2 * (n - 1 - j) + 1] = 0.0;
                }
                fft_.exec(a, b);
                for (std::size_t k = 0; k < n; ++k) {
                    const double c = rot_[2 * k], s = rot_[2 * k + 1];
                    out[k] = 2.0 * (b[2 * k] * c + b[2 * k + 1] * s);
                }
                break;
            }
            case Kind::redft01: {
                // V_k = e^{i pi k/2n} (x_k - i x_{n-k}), x_n = 0; v = IDFT(V);
                // Y_{2p} = Re v_p, Y_{2p+1} = Re v_{n-1-p}.
                for (std::size_t k = 0; k < n; ++k) {
                    const double xr = in[k];
                    const double xi = (k == 0) ? 0.0 : -in[n - k];
                    const double c = rot_[2 * k], s = rot_[2 * k + 1];
                    a[2 * k] = xr * c - xi * s;
                    a[2 * k + 1] = xr * s + xi * c;
                }
                fft_.exec(a, b);
                for (std::size_t p = 0; 2 * p < n; ++p) out[2 * p] = b[2 * p];
                for (std::size_t p = 0; 2 * p + 1 < n; ++p) out[2 * p + 1] = b[2 * (n - 1 - p)];
                break;
            }
            case Kind::rodft00: {
                // Odd extension of length N = 2(n+1); Y_{k-1} = -Im A_k.
                const std::size_t big = 2 * (n + 1);
                for (std::size_t l = 0; l < big; ++l) a[2 * l] = a[2 * l + 1] = 0.0;
                for (std::size_t j = 0; j < n; ++j) {
                    a[2 * (j + 1)] = in[j];
                    a[2 * (big - j - 1)] = -in[j];
                }
                fft_.exec(a, b);
                for (std::size_t k = 1; k <= n; ++k) out[k - 1] = -b[2 * k + 1];
                break;
            }
        }
    }

  private:
    Kind kind_ = Kind::redft10;
    std::size_t n_ = 0;
    Fft fft_;
    std::vector<double> rot_;
};

} // namespace dctp::r2r
