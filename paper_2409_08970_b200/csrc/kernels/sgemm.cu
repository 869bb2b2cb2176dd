// Progressive DCT+ in fp32 as one dense SGEMM (SIMT FFMA), sm_100a.
//
// With c_p = n every member r of a PrunedEnsemblePlan is the full n x n
// orthonormal basis X_r (fast_transform.hpp:355-366 evaluates it as T_r on
// the DCT coefficients), and set 0 is the DCT itself.  For small n
// (n <= 256) the whole forward_all is therefore
//
//     out[b, :] = x[b, :] * G,    G = [D^T | X_1 | ... | X_K]   (n x (K+1) n)
//
// a single GEMM whose B operand (<= 4.5 MB fp32, built on the host in double
// and rounded once) stays in L2, and whose output is exactly the
// [batch][K+1][n] layout.  No DCT pass, no scatter, no per-entry division.
//
// Classic register-tiled SGEMM: CTA tile 128 x 128, BK = 16, 256 threads with
// 8 x 8 outputs each (two 4 x 4 quadrants 64 apart), A transposed into shared
// memory through registers, B copied as float4, both double-buffered with the
// next tile's global loads in flight during the FMAs.  Per k a warp issues 4
// LDS.128 (the A ones broadcast) for 64 FFMA, so the FMA pipe, not shared
// memory, bounds it.
#include <cstdint>

#include "kernels/common.cuh"
#include "kernels/launch.hpp"

namespace dctp::dev {
namespace {

constexpr int BM = 128, BN = 128, BK = 16, kThreads = 256, LDA_S = BM + 4;

__global__ void __launch_bounds__(kThreads, 2)
sgemm_rows_kernel(const float* __restrict__ A, int lda, const float* __restrict__ B, int ldb, float* __restrict__ C,
                  std::size_t ldc, std::size_t M, int N, int K, int* flag, const int* __restrict__ col_map) {
    __shared__ __align__(16) float As[2][BK][LDA_S];
    __shared__ __align__(16) float Bs[2][BK][BN];
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    const int n0 = blockIdx.x * BN; // column tiles vary fastest: CTAs sharing A rows run together
    const std::size_t m0 = static_cast<std::size_t>(blockIdx.y) * BM;

    float4 ra[2], rb[2];
    auto gload = [&](int k0) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const std::size_t m = m0 + tid / 4 + 64 * i;
            ra[i] = m < M ? *reinterpret_cast<const float4*>(A + m * lda + k0 + (tid % 4) * 4)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
            const int kb = tid / 32 + 8 * i, c = n0 + (tid % 32) * 4;
            rb[i] = c < N ? *reinterpret_cast<const float4*>(B + static_cast<std::size_t>(k0 + kb) * ldb + c)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int r = tid / 4 + 64 * i, kq = (tid % 4) * 4;
            As[buf][kq + 0][r] = ra[i].x;
            As[buf][kq + 1][r] = ra[i].y;
            As[buf][kq + 2][r] = ra[i].z;
            As[buf][kq + 3][r] = ra[i].w;
            *reinterpret_cast<float4*>(&Bs[buf][tid / 32 + 8 * i][(tid % 32) * 4]) = rb[i];
        }
    };

    // acc2[i][p] holds columns 2p, 2p+1 of row i: packed FFMA2 halves the
    // issue slots of the FMA stream (the kernel was issue-bound)
    unsigned long long acc2[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) acc2[i][p] = 0ull;

    gload(0);
    sstore(0);
    __syncthreads();
    for (int k0 = 0; k0 < K; k0 += BK) {
        const int buf = (k0 / BK) & 1;
        const bool more = k0 + BK < K;
        if (more) gload(k0 + BK);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const unsigned long long b2[4] = {ptx::pack2(b0.x, b0.y), ptx::pack2(b0.z, b0.w), ptx::pack2(b1.x, b1.y),
                                              ptx::pack2(b1.z, b1.w)};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const unsigned long long aa = ptx::pack2(a[i], a[i]);
#pragma unroll
                for (int p = 0; p < 4; ++p) ptx::ffma2(acc2[i][p], aa, b2[p]);
            }
        }
        if (more) sstore(buf ^ 1); // that buffer was last read before the previous barrier
        __syncthreads();
    }

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) ptx::unpack2(acc2[i][p], acc[i][2 * p], acc[i][2 * p + 1]);
    bool bad = false;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const std::size_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
        if (m >= M) continue;
        float* crow = C + m * ldc;
        const int c0 = n0 + tx * 4, c1 = n0 + 64 + tx * 4;
        if (col_map) { // scattered output slots; every value is checked
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int c = (q < 4 ? c0 : c1) + (q & 3);
                if (c < N) {
                    crow[__ldg(col_map + c)] = acc[i][q];
                    bad |= !isfinite(acc[i][q]);
                }
            }
            continue;
        }
        if (c0 < N) *reinterpret_cast<float4*>(crow + c0) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        if (c1 < N) *reinterpret_cast<float4*>(crow + c1) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
        // column 0 is set 0's DC coefficient, sum(x)/sqrt(n): any non-finite input shows there
        if (c0 == 0) bad |= !isfinite(acc[i][0]);
    }
    if (bad) atomicOr(flag, 1);
}

} // namespace

bool sgemm_rows_supported(int K, int N, int lda, int ldb, std::size_t ldc, const void* A, const void* B, const void* C) {
    const auto al = [](const void* p) { return reinterpret_cast<std::uintptr_t>(p) % 16 == 0; };
    return K % BK == 0 && N % 4 == 0 && lda % 4 == 0 && ldb % 4 == 0 && ldc % 4 == 0 && al(A) && al(B) && al(C);
}

cudaError_t sgemm_rows(const float* A, int lda, const float* B, int ldb, float* C, std::size_t ldc, std::size_t M,
                       int N, int K, int* flag, cudaStream_t stream, const int* col_map) {
    if (M == 0 || N == 0) return cudaSuccess;
    if (!sgemm_rows_supported(K, N, lda, ldb, col_map ? 4 : ldc, A, B, col_map ? B : C)) return cudaErrorInvalidValue;
    constexpr std::size_t kMaxRows = std::size_t{65535} * BM; // gridDim.y limit
    for (std::size_t r0 = 0; r0 < M; r0 += kMaxRows) {
        const std::size_t rows = M - r0 < kMaxRows ? M - r0 : kMaxRows;
        dim3 grid(static_cast<unsigned>((N + BN - 1) / BN), static_cast<unsigned>((rows + BM - 1) / BM));
        sgemm_rows_kernel<<<grid, kThreads, 0, stream>>>(A + r0 * lda, lda, B, ldb, C + r0 * ldc, ldc, rows, N, K,
                                                         flag, col_map);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

} // namespace dctp::dev
