// Per-graph setup on the GPU: the secular-equation roots and the column
// normalisers of the rank-one update, one root per thread.
//
// Reference: secular_eigenvalues / solve_secular_bracket / secular_eval and
// normalizers (proj/include/dctplus/spectral.hpp:149-233, 297-315), restated
// op for op on the host in host/setup.hpp (secular_value, secular_root,
// normalisers).  This file repeats those operations in the same order: the
// sums run sequentially over j, IEEE division and square root, and the file
// is compiled with -fmad=false (_build.py), so every root and normaliser is
// bit-identical to the host restatement and hence to the reference
// (tests/test_gpu_parity.py::test_gpu_setup_bit_identical).  At n = 8192 the
// host spends ~0.8 s of its 1.2 s setup here (8 threads); the GPU ~ms.
#include <cfloat>

#include "kernels/common.cuh"
#include "kernels/launch.hpp"

namespace dctp::dev {
namespace {

struct Value {
    double f, df, scale;
};

__device__ __forceinline__ Value secular_value(const double* __restrict__ lam, const double* __restrict__ z, int k,
                                               double rho, double x) {
    double sum = 0.0, dsum = 0.0, asum = 0.0;
    for (int j = 0; j < k; ++j) {
        const double gap = __ldg(lam + j) - x;
        const double zj = __ldg(z + j);
        const double term = zj * zj / gap;
        sum += term;
        dsum += term / gap;
        asum += fabs(term);
    }
    return {1.0 + rho * sum, rho * dsum, 1.0 + fabs(rho) * asum};
}

/// Safeguarded Newton on the bracket of root r (host/setup.hpp secular_root):
/// midpoint start, a forced bisection every fourth step or whenever Newton
/// leaves the bracket; at most 200 iterations (status 1 otherwise).
__global__ void secular_roots_kernel(const double* __restrict__ lam, const double* __restrict__ z, int k, double rho,
                                     double zz, double* __restrict__ mu, int* status) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= k) return;
    double lo, hi;
    if (rho > 0.0) {
        lo = lam[r];
        hi = (r + 1 < k) ? lam[r + 1] : lam[k - 1] + rho * zz;
    } else {
        lo = (r == 0) ? lam[0] + rho * zz : lam[r - 1];
        hi = lam[r];
    }
    const double dir = (rho > 0.0) ? 1.0 : -1.0;
    const double ulp4 = 4.0 * DBL_EPSILON;
    const double tiny = DBL_MIN;
    double x = 0.5 * (lo + hi);
    for (int it = 0; it < 200; ++it) {
        const Value e = secular_value(lam, z, k, rho, x);
        if (fabs(e.f) <= 1e-15 * e.scale) {
            mu[r] = x;
            return;
        }
        if (dir * e.f < 0.0)
            lo = x;
        else
            hi = x;
        if (hi - lo <= ulp4 * (fabs(lo) + fabs(hi) + tiny)) {
            mu[r] = 0.5 * (lo + hi);
            return;
        }
        double next = x - e.f / e.df;
        if (!(next > lo && next < hi) || e.df == 0.0 || (it % 4) == 3) next = 0.5 * (lo + hi);
        x = next;
    }
    atomicOr(status, 1);
}

/// a_i = (sum_j (z_j / (mu_i - lambda_j))^2)^(-1/2) over z_j != 0 (host/setup.hpp
/// normalisers); status 2: mu/lambda collision, 4: degenerate column.
__global__ void normalisers_kernel(const double* __restrict__ lam, const double* __restrict__ z, int m,
                                   const double* __restrict__ mu, int k, double* __restrict__ a, int* status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    const double x = mu[i];
    double s = 0.0;
    for (int j = 0; j < m; ++j) {
        const double zj = __ldg(z + j);
        const double d = x - __ldg(lam + j);
        if (d == 0.0 && zj != 0.0) {
            atomicOr(status, 2);
            return;
        }
        if (zj != 0.0) s += (zj / d) * (zj / d);
    }
    if (!(s > 0.0) || !isfinite(s)) {
        atomicOr(status, 4);
        return;
    }
    a[i] = 1.0 / sqrt(s);
}

/// One CTA per column: peak = max |x_i|, then the lowest i with |x_i| >=
/// peak (1 - 1e-12) (host/setup.hpp sign_of_column).
__global__ void column_signs_kernel(const double* __restrict__ xt, std::size_t ld, int n, double* __restrict__ sign) {
    __shared__ double red[32];
    __shared__ int ired[32];
    const double* x = xt + static_cast<std::size_t>(blockIdx.x) * ld;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double peak = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) peak = fmax(peak, fabs(x[i]));
    for (int o = 16; o > 0; o >>= 1) peak = fmax(peak, __shfl_xor_sync(0xffffffffu, peak, o));
    if (lane == 0) red[warp] = peak;
    __syncthreads();
    peak = 0.0;
    for (int w = 0; w < nw; ++w) peak = fmax(peak, red[w]);
    if (peak == 0.0) {
        if (threadIdx.x == 0) sign[blockIdx.x] = 1.0;
        return;
    }
    const double thr = peak * (1.0 - 1e-12);
    int first = n;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        if (fabs(x[i]) >= thr) {
            first = i;
            break;
        }
    for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    if (lane == 0) ired[warp] = first;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 0; w < nw; ++w) first = min(first, ired[w]);
        sign[blockIdx.x] = (first < n && x[first] < 0.0) ? -1.0 : 1.0;
    }
}

} // namespace

cudaError_t column_signs_gpu(const double* xt, std::size_t ld, int n, int cols, double* sign, cudaStream_t stream) {
    if (cols <= 0) return cudaSuccess;
    column_signs_kernel<<<cols, 256, 0, stream>>>(xt, ld, n, sign);
    return cudaGetLastError();
}

cudaError_t secular_roots_gpu(const double* lam, const double* z, int k, double rho, double zz, double* mu,
                              int* status, cudaStream_t stream) {
    if (k <= 0) return cudaSuccess;
    constexpr int threads = 128;
    secular_roots_kernel<<<(k + threads - 1) / threads, threads, 0, stream>>>(lam, z, k, rho, zz, mu, status);
    return cudaGetLastError();
}

cudaError_t normalisers_gpu(const double* lam, const double* z, int m, const double* mu, int k, double* a,
                            int* status, cudaStream_t stream) {
    if (k <= 0) return cudaSuccess;
    constexpr int threads = 128;
    normalisers_kernel<<<(k + threads - 1) / threads, threads, 0, stream>>>(lam, z, m, mu, k, a, status);
    return cudaGetLastError();
}

} // namespace dctp::dev
