// Pruned progressive mode of PrunedEnsemblePlan (c_p < n), sm_100a.
//
// fast_transform.hpp:396-439.  Per signal s with DCT coefficients sd:
//   q = sum_i (s_i - s_{i+1})^2                     (path_quadratic_form, :24-31)
//   q <= threshold: the signal is "pruned":
//     set 0 keeps sd[0, c_p), the rest is zeroed, bound_0 = ||sd[c_p, n)||;
//     member r: y = UL_r sd[0, c_p) in its first c_p slots (rest 0),
//               bound_r = bound_0 + ||HL_r sd[0, c_p)||,
//     with [UL_r; HL_r] = T_r[:, 0:c_p] (n x c_p, host-built like :355-366);
//   otherwise every member is computed in full and the bounds are 0.
//
// The batch first goes through the full progressive path (every set of every
// signal); this kernel then rewrites the pruned signals in place.  One CTA per
// 16 signals: warps compute q, the tail norm and the kept coefficients, then
// all threads sweep (signal, slot) pairs member by member, each block row
// dotted with the signal's c_p coefficients (the n x c_p block is read from
// L1/L2 and reused by the CTA's 16 signals), leak norms accumulated in shared
// memory.
#include <algorithm>
#include <cmath>

#include "kernels/common.cuh"
#include "kernels/launch.hpp"

namespace dctp::dev {
namespace {

constexpr int kThreads = 256, kSig = 16, kWarps = kThreads / 32;

template <class T>
__global__ void __launch_bounds__(kThreads)
ensemble_prune_kernel(const T* __restrict__ in, T* __restrict__ out, const T* __restrict__ blocks, int n, int cp,
                      int members, double threshold, std::size_t batch, T* __restrict__ bounds,
                      unsigned char* __restrict__ pruned_flags) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* sd = reinterpret_cast<double*>(smem_raw); // kSig x cp kept coefficients
    __shared__ double tail[kSig], leak[kSig];
    __shared__ int pr[kSig];
    const int sets = members + 1;
    const std::size_t b0 = static_cast<std::size_t>(blockIdx.x) * kSig;
    const int nsig = static_cast<int>(min(static_cast<std::size_t>(kSig), batch - b0));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    for (int s = warp; s < kSig; s += kWarps) {
        if (s >= nsig) {
            if (lane == 0) pr[s] = 0;
            continue;
        }
        const std::size_t b = b0 + s;
        const T* x = in + b * n;
        double q = 0.0;
        for (int i = lane; i + 1 < n; i += 32) {
            const double d = static_cast<double>(x[i]) - static_cast<double>(x[i + 1]);
            q += d * d;
        }
        T* o0 = out + b * sets * n;
        double t2 = 0.0;
        for (int j = cp + lane; j < n; j += 32) t2 += static_cast<double>(o0[j]) * static_cast<double>(o0[j]);
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) {
            q += __shfl_xor_sync(0xffffffffu, q, m);
            t2 += __shfl_xor_sync(0xffffffffu, t2, m);
        }
        const bool p = q <= threshold;
        if (p) {
            for (int j = lane; j < cp; j += 32) sd[s * cp + j] = static_cast<double>(o0[j]);
            for (int j = cp + lane; j < n; j += 32) o0[j] = T(0);
        }
        if (lane == 0) {
            pr[s] = p ? 1 : 0;
            tail[s] = p ? sqrt(t2) : 0.0;
            leak[s] = 0.0;
            if (pruned_flags) pruned_flags[b] = p ? 1 : 0;
            if (bounds) bounds[b * sets] = p ? static_cast<T>(sqrt(t2)) : T(0);
        }
    }
    __syncthreads();
    bool any = false;
    for (int s = 0; s < nsig; ++s) any |= pr[s] != 0;
    if (!any) {
        // full branch for every signal here: bounds are 0
        if (bounds)
            for (int t = tid; t < nsig * members; t += kThreads) bounds[(b0 + t / members) * sets + 1 + t % members] = T(0);
        return;
    }
    for (int r = 0; r < members; ++r) {
        const T* blk = blocks + static_cast<std::size_t>(r) * n * cp; // n x cp, row = output slot
        for (int t = tid; t < nsig * n; t += kThreads) {
            const int s = t / n, i = t - s * n;
            if (!pr[s]) continue;
            const T* row = blk + static_cast<std::size_t>(i) * cp;
            const double* v = sd + s * cp;
            double z = 0.0;
            for (int j = 0; j < cp; ++j) z = fma(static_cast<double>(row[j]), v[j], z);
            T* o = out + ((b0 + s) * sets + 1 + r) * n;
            if (i < cp) {
                o[i] = static_cast<T>(z);
            } else {
                o[i] = T(0);
                atomicAdd(&leak[s], z * z);
            }
        }
        __syncthreads();
        if (tid < nsig) {
            if (bounds) bounds[(b0 + tid) * sets + 1 + r] = pr[tid] ? static_cast<T>(tail[tid] + sqrt(leak[tid])) : T(0);
            leak[tid] = 0.0;
        }
        __syncthreads();
    }
}

/// c_p = n: nothing to rewrite; flags from the quadratic form, bounds 0.
template <class T>
__global__ void __launch_bounds__(kThreads)
ensemble_flags_kernel(const T* __restrict__ in, int n, int sets, double threshold, std::size_t batch,
                      T* __restrict__ bounds, unsigned char* __restrict__ pruned_flags) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const std::size_t b = static_cast<std::size_t>(blockIdx.x) * kWarps + warp;
    if (b >= batch) return;
    const T* x = in + b * n;
    double q = 0.0;
    for (int i = lane; i + 1 < n; i += 32) {
        const double d = static_cast<double>(x[i]) - static_cast<double>(x[i + 1]);
        q += d * d;
    }
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) q += __shfl_xor_sync(0xffffffffu, q, m);
    if (bounds)
        for (int r = lane; r < sets; r += 32) bounds[b * sets + r] = T(0);
    if (lane == 0 && pruned_flags) pruned_flags[b] = q <= threshold ? 1 : 0;
}

} // namespace

template <class T>
cudaError_t ensemble_prune(const T* in, T* out, const T* blocks, std::size_t n, std::size_t cp, int members,
                           double threshold, std::size_t batch, T* bounds, unsigned char* pruned,
                           cudaStream_t stream) {
    if (batch == 0) return cudaSuccess;
    if (cp >= n) {
        if (!bounds && !pruned) return cudaSuccess;
        const unsigned grid = static_cast<unsigned>((batch + kWarps - 1) / kWarps);
        ensemble_flags_kernel<T><<<grid, kThreads, 0, stream>>>(in, static_cast<int>(n), members + 1, threshold,
                                                                batch, bounds, pruned);
        return cudaGetLastError();
    }
    const std::size_t smem = kSig * cp * sizeof(double);
    if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(ensemble_prune_kernel<T>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    const unsigned grid = static_cast<unsigned>((batch + kSig - 1) / kSig);
    ensemble_prune_kernel<T><<<grid, kThreads, smem, stream>>>(in, out, blocks, static_cast<int>(n),
                                                               static_cast<int>(cp), members, threshold, batch,
                                                               bounds, pruned);
    return cudaGetLastError();
}

template cudaError_t ensemble_prune<double>(const double*, double*, const double*, std::size_t, std::size_t, int,
                                            double, std::size_t, double*, unsigned char*, cudaStream_t);
template cudaError_t ensemble_prune<float>(const float*, float*, const float*, std::size_t, std::size_t, int,
                                           double, std::size_t, float*, unsigned char*, cudaStream_t);

} // namespace dctp::dev

namespace dctp::dev {
namespace {

/// rdo_select (fast_transform.hpp:472-496) for a batch: per signal the set
/// with the smallest l1 norm (ties to the lower index), copied out.
template <class T>
__global__ void __launch_bounds__(kThreads)
rdo_select_kernel(const T* __restrict__ coeffs, int n, int sets, std::size_t batch, T* __restrict__ chosen,
                  int* __restrict__ index) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const std::size_t b = static_cast<std::size_t>(blockIdx.x) * kWarps + warp;
    if (b >= batch) return;
    const T* c = coeffs + b * sets * n;
    double best = 0.0;
    int arg = 0;
    for (int r = 0; r < sets; ++r) {
        double l1 = 0.0;
        for (int i = lane; i < n; i += 32) l1 += fabs(static_cast<double>(c[r * n + i]));
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, m);
        if (r == 0 || l1 < best) {
            best = l1;
            arg = r;
        }
    }
    if (chosen)
        for (int i = lane; i < n; i += 32) chosen[b * n + i] = c[arg * n + i];
    if (lane == 0 && index) index[b] = arg;
}

} // namespace

template <class T>
cudaError_t rdo_select_rows(const T* coeffs, std::size_t n, int sets, std::size_t batch, T* chosen, int* index,
                            cudaStream_t stream) {
    if (batch == 0) return cudaSuccess;
    const unsigned grid = static_cast<unsigned>((batch + kWarps - 1) / kWarps);
    rdo_select_kernel<T><<<grid, kThreads, 0, stream>>>(coeffs, static_cast<int>(n), sets, batch, chosen, index);
    return cudaGetLastError();
}

template cudaError_t rdo_select_rows<double>(const double*, std::size_t, int, std::size_t, double*, int*,
                                             cudaStream_t);
template cudaError_t rdo_select_rows<float>(const float*, std::size_t, int, std::size_t, float*, int*, cudaStream_t);

} // namespace dctp::dev
