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
#include <cstdint>
#include <type_traits>

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

// ---- fp32: register-tiled SGEMM form ---------------------------------------------
//
// The fp32 Cauchy stage as a SIMT SGEMM (the tiling of kernels/sgemm.cu:
// 128 x 128 x 16 tiles, 256 threads, 8 x 8 outputs each, double-buffered
// shared memory): A rows come from global memory (float4 when the inputs are
// already compacted, a gather through src[] otherwise) one chunk ahead in
// registers; the B chunk, rscale[r] / (x_r - y_c), is generated straight into
// the next shared buffer from fp64 gaps (one fp64 subtract, one MUFU rcp per
// entry, amortised over 128 signals).  The 64 x 64 tile kernel above is
// shared-memory bound at ~25% of FFMA peak; this one is FMA bound.
constexpr int SBM = 128, SBN = 128, SBK = 16, SLDA = SBM + 4;

__global__ void __launch_bounds__(kThreads, 2)
cauchy_sgemm_kernel(const float* __restrict__ in, std::size_t ld_in, float* __restrict__ out, std::size_t ld_out,
                    const CauchyStage* __restrict__ stages, std::size_t batch, int* flag, int vec4) {
    __shared__ __align__(16) float As[2][SBK][SLDA];
    __shared__ __align__(16) float Bs[2][SBK][SBN];
    __shared__ double ys[SBN];
    const CauchyStage st = stages[blockIdx.z];
    const int c0 = blockIdx.y * SBN;
    if (c0 >= st.cols) return;
    const std::size_t b0 = static_cast<std::size_t>(blockIdx.x) * SBM;
    const float* rscale = static_cast<const float*>(st.rscale);
    const float* cscale = static_cast<const float*>(st.cscale);
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    for (int c = tid; c < SBN; c += kThreads) ys[c] = c0 + c < st.cols ? st.y[c0 + c] : 0.0;
    const bool use_vec = st.src_contig && vec4;

    float ra[8];
    bool bad = false;
    auto gload = [&](int r0) {
        if (use_vec) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const std::size_t b = b0 + tid / 4 + 64 * i;
                const int r = r0 + (tid % 4) * 4;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (b < batch) {
                    if (r + 3 < st.rows) {
                        v = *reinterpret_cast<const float4*>(in + b * ld_in + r);
                    } else {
                        const float* p = in + b * ld_in;
                        v.x = r < st.rows ? p[r] : 0.f;
                        v.y = r + 1 < st.rows ? p[r + 1] : 0.f;
                        v.z = r + 2 < st.rows ? p[r + 2] : 0.f;
                    }
                }
                ra[4 * i + 0] = v.x;
                ra[4 * i + 1] = v.y;
                ra[4 * i + 2] = v.z;
                ra[4 * i + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int e = tid + kThreads * i, kk = e % SBK, bb = e / SBK;
                const int r = r0 + kk;
                const std::size_t b = b0 + bb;
                ra[i] = (r < st.rows && b < batch) ? in[b * ld_in + st.src[r]] : 0.f;
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) bad |= !finite_val(ra[i]);
    };
    auto sstore_a = [&](int buf) {
        if (use_vec) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int row = tid / 4 + 64 * i, kq = (tid % 4) * 4;
#pragma unroll
                for (int j = 0; j < 4; ++j) As[buf][kq + j][row] = ra[4 * i + j];
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int e = tid + kThreads * i;
                As[buf][e % SBK][e / SBK] = ra[i];
            }
        }
    };
    auto gen_b = [&](int r0, int buf) {
#pragma unroll
        for (int i = 0; i < (SBK * SBN) / kThreads; ++i) {
            const int e = tid + kThreads * i, kk = e / SBN, cc = e % SBN;
            const int r = r0 + kk;
            Bs[buf][kk][cc] = (r < st.rows && c0 + cc < st.cols)
                                  ? rscale[r] * __frcp_rn(static_cast<float>(st.x[r] - ys[cc]))
                                  : 0.f;
        }
    };

    unsigned long long acc2[8][4]; // columns 2p, 2p+1 of row i, packed for FFMA2 (see sgemm.cu)
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) acc2[i][p] = 0ull;

    __syncthreads(); // ys
    gload(0);
    sstore_a(0);
    gen_b(0, 0);
    __syncthreads();
    for (int r0 = 0; r0 < st.rows; r0 += SBK) {
        const int buf = (r0 / SBK) & 1;
        const bool more = r0 + SBK < st.rows;
        if (more) gload(r0 + SBK);
#pragma unroll
        for (int kk = 0; kk < SBK; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
            const float4 q0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
            const float4 q1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const unsigned long long b2[4] = {ptx::pack2(q0.x, q0.y), ptx::pack2(q0.z, q0.w), ptx::pack2(q1.x, q1.y),
                                              ptx::pack2(q1.z, q1.w)};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const unsigned long long aa = ptx::pack2(a[i], a[i]);
#pragma unroll
                for (int p = 0; p < 4; ++p) ptx::ffma2(acc2[i][p], aa, b2[p]);
            }
        }
        if (more) {
            sstore_a(buf ^ 1);
            gen_b(r0 + SBK, buf ^ 1);
        }
        __syncthreads();
    }
    if (bad) atomicOr(flag, 1);

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) ptx::unpack2(acc2[i][p], acc[i][2 * p], acc[i][2 * p + 1]);
    int dst[8];
    float cs[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int c = c0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
        dst[j] = c < st.cols ? st.dst[c] : -1;
        cs[j] = c < st.cols ? cscale[c] : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const std::size_t b = b0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
        if (b >= batch) continue;
        float* orow = out + b * ld_out + st.out_offset;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (dst[j] >= 0) orow[dst[j]] = cs[j] * acc[i][j];
    }
}

} // namespace

template <class T>
cudaError_t cauchy_rows(const T* in, std::size_t ld_in, T* out, std::size_t ld_out,
                        const CauchyStage* stages_dev, int num_stages, int max_rows, int max_cols,
                        std::size_t batch, int* flag, cudaStream_t stream) {
    if (batch == 0 || num_stages == 0 || max_cols == 0) return cudaSuccess;
    if constexpr (std::is_same_v<T, float>) {
        if (max_rows >= 64) {
            dim3 grid(static_cast<unsigned>((batch + SBM - 1) / SBM), static_cast<unsigned>((max_cols + SBN - 1) / SBN),
                      static_cast<unsigned>(num_stages));
            const int vec4 = reinterpret_cast<std::uintptr_t>(in) % 16 == 0 && ld_in % 4 == 0;
            cauchy_sgemm_kernel<<<grid, kThreads, 0, stream>>>(in, ld_in, out, ld_out, stages_dev, batch, flag, vec4);
            return cudaGetLastError();
        }
    }
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
