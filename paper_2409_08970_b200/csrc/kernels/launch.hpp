// Host-visible launchers of the sm_100a kernels (no CUDA types leak beyond
// cudaStream_t).  Implemented in dct.cu / cauchy.cu; called by plan.cpp.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime_api.h>

namespace dctp::dev {

/// Twiddle tables of one power-of-two length n (N = n/2 complex points),
/// interleaved (cos, sin) in T, device-resident.
template <class T>
struct Twiddles {
    const T* fft = nullptr;   // e^{-2 pi i k / N},      k < N/2
    const T* split = nullptr; // e^{-2 pi i k / n},      k < N
    const T* rot = nullptr;   // e^{-i pi k / (2n)},     k <= N
    const T* cos4n = nullptr; // cos(pi m / (2n)), m < 4n (direct kernels, any n)
};

/// Index/value list for a scattered copy dst[b*ld + to[e]] = sign[e] * src[from[e]].
template <class T>
struct Emit {
    const int* to = nullptr;
    const int* from = nullptr;
    const T* sign = nullptr;
    int count = 0;
};

/// Forward DCT-II of `batch` rows of length n (orthonormal, U^T s):
///   hat[b*ld_hat + k]     = shat_k          (if hat != nullptr)
///   out[b*ld_out + to[e]] = sign[e] * shat_{from[e]}   for each emit entry
/// Non-finite input samples set *flag (the domain_error of check_signal).
template <class T>
cudaError_t dct2_rows(const T* in, std::size_t ld_in, T* hat, std::size_t ld_hat, T* out,
                      std::size_t ld_out, Emit<T> emit, std::size_t n, std::size_t batch,
                      Twiddles<T> tw, int* flag, cudaStream_t stream);

/// Inverse (DCT-III, orthonormal, U d) of rows d; before the transform
///   d[to[e]] = sign[e] * p[b*ld_p + from[e]]  (the pass-through slots).
template <class T>
cudaError_t idct_rows(const T* d, std::size_t ld_d, const T* p, std::size_t ld_p, Emit<T> emit,
                      T* out, std::size_t ld_out, std::size_t n, std::size_t batch,
                      Twiddles<T> tw, int* flag, cudaStream_t stream);

/// One Cauchy stage (SIMT, entries generated on the fly from fp64 gaps):
///   out[b*ld_out + dst[c]] = cscale[c] * sum_r rscale[r] * in[b*ld_in + src[r]] / (x[r] - y[c])
struct CauchyStage {
    const int* src;       // R
    const double* x;      // R
    const void* rscale;   // R, T
    const int* dst;       // C
    const double* y;      // C
    const void* cscale;   // C, T
    int rows;             // R
    int cols;             // C
    std::int64_t out_offset; // element offset of this stage's output within a row block
};

template <class T>
cudaError_t cauchy_rows(const T* in, std::size_t ld_in, T* out, std::size_t ld_out,
                        const CauchyStage* stages_dev, int num_stages, int max_rows, int max_cols,
                        std::size_t batch, int* flag, cudaStream_t stream);

/// Constants of the fused small-plan forward kernel (fused_small.cu).
struct SmallPlanDev {
    const double* lam_kept;  // K
    const double* z_kept;    // K
    const double* nu;        // A (secular roots, ascending)
    const double* act_scale; // A (sigma * a of the root's slot)
    const int* act_slot;     // A
    const double* tmat;      // A x K: T[c][k] = sigma_c a_c z_k / (lambda_k - mu_c)
    const int* kept_idx;     // K: DCT index of each kept coefficient
    const int* pass_src;     // n - K: DCT index of each pass-through coefficient
    const int* pass_slot;    // n - K: its output slot
    const int* pass_neg;     // n - K: 1 if sigma of that slot is -1
    const double* fft_tw;    // N = n/2 complex e^{-2 pi i m / N}
    const double* split_tw;  // N complex e^{-2 pi i k / n}
    const double* rot_tw;    // N+1 complex e^{-i pi k / 2n}
    int n, K, A;
    int debug; // development knob (DCTP_DEBUG_MODE): 1 = skip the DCT work, 2 = skip the DMMA work
};

bool fused_small_supported(std::size_t n, int K, int A);
cudaError_t fused_small_forward(const double* in, double* out, std::size_t batch, const SmallPlanDev& P, int* flag,
                                int num_sms, cudaStream_t stream);

} // namespace dctp::dev
