// Cauchy stage of DCT+ (the diag(z) C(lambda, mu) diag(sigma a) factor),
// generic SIMT form, sm_100a.
//
//   out[b, dst[c]] = cscale[c] * sum_r rscale[r] * in[b, src[r]] / (x[r] - y[c])
//
// Forward (fast_transform.hpp:163-190 / the dense route :199-209):
//   src = kept DCT indices, rscale = z, x = lambda_kept, y = mu_active,
//   cscale = sigma*a, dst = active output slots.
// Inverse (:218-255): src = active slots, rscale = sigma*a, x = mu_active,
//   y = lambda_kept, cscale = -z, dst = kept DCT indices.
// Progressive mode (:396-439, c_p = n): blockIdx.z walks the K members.
//
// The Cauchy entries are never materialised in HBM: every CTA generates its
// BK x BN tile in shared memory from fp64 gaps and
// reuses each entry across BM signals, so the per-entry division costs
// ~BN*BK/(BM*BN*BK/(TM*TN)) of the FMA work.
#include <algorithm>

#include "kernels/common.cuh"
#include "kernels/launch.hpp"

namespace dctp::dev {
namespace {

constexpr int kThreads = 256;
constexpr int BK = 16;

template <class T, int BM, int BN>
__global__ void __launch_bounds__(kThreads)
cauchy_tile_kernel(const T* __restrict__ in, std::size_t ld_in, T* __restrict__ out, std::size_t ld_out,
                   const CauchyStage* __restrict__ stages, std::size_t batch, int* flag) {
    constexpr int TM = BM / 16, TN = BN / 16;
    const CauchyStage st = stages[blockIdx.z];
    const int c0 = blockIdx.y * BN;
    if (c0 >= st.cols) return;
    const std::size_t b0 = static_cast<std::size_t>(blockIdx.x) * BM;
    const T* rscale = static_cast<const T*>(st.rscale);
    const T* cscale = static_cast<const T*>(st.cscale);

    __shared__ T As[BK][BM + 1];
    __shared__ T Cs[BK][BN + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    T acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

    bool bad = false;
    for (int r0 = 0; r0 < st.rows; r0 += BK) {
#pragma unroll
        for (int q = 0; q < (BM * BK) / kThreads; ++q) {
            const int e = threadIdx.x + kThreads * q;
            const int kk = e % BK, bb = e / BK;
            const int r = r0 + kk;
            const std::size_t b = b0 + bb;
            T v = T(0);
            if (r < st.rows && b < batch) {
                v = in[b * ld_in + st.src[r]];
                bad |= !finite_val(v);
                v *= rscale[r];
            }
            As[kk][bb] = v;
        }
#pragma unroll
        for (int q = 0; q < (BN * BK) / kThreads; ++q) {
            const int e = threadIdx.x + kThreads * q;
            const int kk = e / BN, cc = e % BN;
            const int r = r0 + kk, c = c0 + cc;
            Cs[kk][cc] = (r < st.rows && c < st.cols) ? cauchy_entry<T>(st.x[r], st.y[c]) : T(0);
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            T a[TM], bv[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < TN; ++j) bv[j] = Cs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
    if (bad) atomicOr(flag, 1);
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const std::size_t b = b0 + ty + 16 * i;
        if (b >= batch) continue;
        T* orow = out + b * ld_out + st.out_offset;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int c = c0 + tx + 16 * j;
            if (c < st.cols) orow[st.dst[c]] = cscale[c] * acc[i][j];
        }
    }
}

} // namespace

template <class T>
cudaError_t cauchy_rows(const T* in, std::size_t ld_in, T* out, std::size_t ld_out,
                        const CauchyStage* stages_dev, int num_stages, int max_rows, int max_cols,
                        std::size_t batch, int* flag, cudaStream_t stream) {
    (void)max_rows;
    if (batch == 0 || num_stages == 0 || max_cols == 0) return cudaSuccess;
    constexpr int BM = 64, BN = 64;
    dim3 grid(static_cast<unsigned>((batch + BM - 1) / BM), static_cast<unsigned>((max_cols + BN - 1) / BN),
              static_cast<unsigned>(num_stages));
    cauchy_tile_kernel<T, BM, BN><<<grid, kThreads, 0, stream>>>(in, ld_in, out, ld_out, stages_dev, batch, flag);
    return cudaGetLastError();
}

template cudaError_t cauchy_rows<double>(const double*, std::size_t, double*, std::size_t, const CauchyStage*, int,
                                         int, int, std::size_t, int*, cudaStream_t);
template cudaError_t cauchy_rows<float>(const float*, std::size_t, float*, std::size_t, const CauchyStage*, int,
                                        int, int, std::size_t, int*, cudaStream_t);

} // namespace dctp::dev
