// ORACLE TEST INFRASTRUCTURE — never linked into the product.
//
// FFTW3 API stand-in for building the reference headers in this image, where
// FFTW3 is absent (proj/CMakeLists.txt:12-13 links an
// unpinned system libfftw3).  Only the subset the reference calls is provided:
//   fftw_plan_r2r_1d / fftw_execute_r2r   trig.hpp:45-53, :96, :106, :112
//   fftw_plan_dft_1d / fftw_execute_dft   nfst.hpp:161-162, :225, :275
//   fftw_alloc_complex / fftw_free        nfst.hpp:37, :47, :59
//   fftw_destroy_plan                     trig.hpp:58, :69; nfst.hpp:167, :175
// The transforms follow FFTW's published kind definitions and are executed by
// paper_2409_08970_b200/csrc/host/r2r.hpp — the one host r2r implementation
// the product's per-graph setup also uses, so z = dct2(v) is bit-identical on
// both sides.  Planner flags are accepted and ignored.
// Plans are immutable; execution is thread-safe (thread_local scratch).
#ifndef DCTP_FFTW_SHIM_FFTW3_H
#define DCTP_FFTW_SHIM_FFTW3_H

#include <cstddef>
#include <cstdlib>
#include <vector>

#include "host/r2r.hpp"

typedef double fftw_complex[2];

typedef enum fftw_r2r_kind_do_not_use_me {
    FFTW_R2HC = 0, FFTW_HC2R = 1, FFTW_DHT = 2,
    FFTW_REDFT00 = 3, FFTW_REDFT01 = 4, FFTW_REDFT10 = 5, FFTW_REDFT11 = 6,
    FFTW_RODFT00 = 7, FFTW_RODFT01 = 8, FFTW_RODFT10 = 9, FFTW_RODFT11 = 10
} fftw_r2r_kind;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_DESTROY_INPUT (1U << 0)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

struct fftw_plan_s {
    bool complex_plan = false;
    dctp::r2r::R2r r2r;
    dctp::r2r::Fft fft;
};
typedef fftw_plan_s* fftw_plan;

inline fftw_plan fftw_plan_r2r_1d(int n, double*, double*, fftw_r2r_kind kind, unsigned) {
    if (n <= 0) return nullptr;
    dctp::r2r::Kind k;
    switch (kind) {
        case FFTW_REDFT10: k = dctp::r2r::Kind::redft10; break;
        case FFTW_REDFT01: k = dctp::r2r::Kind::redft01; break;
        case FFTW_RODFT00: k = dctp::r2r::Kind::rodft00; break;
        default: return nullptr;
    }
    fftw_plan p = new fftw_plan_s;
    p->r2r = dctp::r2r::R2r(k, static_cast<std::size_t>(n));
    return p;
}

inline fftw_plan fftw_plan_dft_1d(int n, fftw_complex*, fftw_complex*, int sign, unsigned) {
    if (n <= 0) return nullptr;
    fftw_plan p = new fftw_plan_s;
    p->complex_plan = true;
    p->fft = dctp::r2r::Fft(static_cast<std::size_t>(n), sign);
    return p;
}

inline void fftw_destroy_plan(fftw_plan p) { delete p; }

namespace dctp_fftw_shim_detail {
inline std::vector<double>& scratch(std::size_t n) {
    thread_local std::vector<double> buf;
    if (buf.size() < n) buf.resize(n);
    return buf;
}
} // namespace dctp_fftw_shim_detail

inline void fftw_execute_r2r(const fftw_plan p, double* in, double* out) {
    const std::size_t len = p->r2r.size();
    std::vector<double>& s = dctp_fftw_shim_detail::scratch(p->r2r.scratch_size() + len);
    // Copy the input first so in == out (allowed by FFTW) stays correct.
    double* tmp = s.data() + p->r2r.scratch_size();
    for (std::size_t i = 0; i < len; ++i) tmp[i] = in[i];
    p->r2r.exec(tmp, out, s.data());
}

inline void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    const std::size_t n = p->fft.size();
    std::vector<double>& s = dctp_fftw_shim_detail::scratch(2 * n);
    const double* src = &in[0][0];
    for (std::size_t i = 0; i < 2 * n; ++i) s[i] = src[i];
    p->fft.exec(s.data(), &out[0][0]);
}

inline fftw_complex* fftw_alloc_complex(std::size_t n) {
    return static_cast<fftw_complex*>(std::aligned_alloc(64, ((n * sizeof(fftw_complex) + 63) / 64) * 64));
}

inline void fftw_free(void* p) { std::free(p); }

#endif
