// Shared device helpers for the DCT+ kernels (sm_100a).
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace dctp::dev {

template <class T>
struct Cplx;
template <>
struct Cplx<double> {
    using type = double2;
};
template <>
struct Cplx<float> {
    using type = float2;
};
template <class T>
using cplx_t = typename Cplx<T>::type;

__device__ __forceinline__ unsigned bit_reverse(unsigned x, int bits) {
    return bits == 0 ? 0u : (__brev(x) >> (32 - bits));
}

__device__ __forceinline__ bool finite_val(double x) { return isfinite(x); }
__device__ __forceinline__ bool finite_val(float x) { return isfinite(x); }

/// Cauchy entry 1/(x - y) with the gap formed in fp64 (SURVEY.md section 0.4:
/// fp32 gaps lose up to 1e-2; fp64 gaps rounded to fp32 entries keep ~1e-6).
template <class T>
__device__ __forceinline__ T cauchy_entry(double x, double y);
template <>
__device__ __forceinline__ double cauchy_entry<double>(double x, double y) {
    return 1.0 / (x - y);
}
template <>
__device__ __forceinline__ float cauchy_entry<float>(double x, double y) {
    return __frcp_rn(static_cast<float>(x - y));
}

inline int ilog2(std::size_t n) {
    int l = 0;
    while ((std::size_t{1} << l) < n) ++l;
    return l;
}

inline bool is_pow2(std::size_t n) { return n != 0 && (n & (n - 1)) == 0; }

} // namespace dctp::dev
