// Signal rows times a stored basis on the fp64 tensor cores (DMMA), sm_100a:
//
//   out[b, c] = sum_k in[b, k] * bt[c, k]          (bt = X^T, row-major, ld_bt)
//
// the batched apply of a rank-k chain (chain.hpp: the composed basis X).  Same
// tiling as the Cauchy DMMA kernel (cauchy_dmma.cu): CTA tile 64 x 128, 8 warps
// of 32 x 32, BK = 32, two CTAs per SM, m8n8k4 fragments from rows padded to 36
// doubles.  Here the B operand is read rather than generated: X^T rows are
// contiguous in k, so A and B chunks are both 16-byte cp.async copies issued
// one chunk ahead; X (<= a few MB for n <= 1024) stays in L2 across the
// batch's row tiles.  fp32 signals are widened while staging (register
// prefetch), so fp32 chains are also accumulated in fp64.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels/common.cuh"
#include "kernels/launch.hpp"

namespace dctp::dev {
namespace {

constexpr int BM = 64, BN = 128, BK = 32, LDS_ = BK + 4;
constexpr int kThreads = 256;
constexpr int WM = 32, WN = 32;
constexpr int MF = WM / 8, NF = WN / 8;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(ptx::smem_addr(smem)), "l"(gmem), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(ptx::smem_addr(smem)), "l"(gmem),
                 "r"(pred ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

template <class T>
__global__ void __launch_bounds__(kThreads, 2)
rows_by_basis_kernel(const T* __restrict__ in, std::size_t ld_in, const double* __restrict__ bt, std::size_t ld_bt,
                     int K, int N, T* __restrict__ out, std::size_t ld_out, std::size_t batch, int* flag, int vec16,
                     const int* __restrict__ col_map, const int* __restrict__ a_map, const T* __restrict__ fold_add,
                     std::size_t ld_add, unsigned kGroup) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* As = reinterpret_cast<double*>(smem_raw); // 2 x BM x LDS_
    double* Bs = As + 2 * BM * LDS_;                  // 2 x BN x LDS_ ([c][k])
    // Grouped tile order: kGroup row tiles at a time sweep every column tile
    // (column fastest within the group), so the CTAs in flight share their A
    // row tiles and each B column tile is read from DRAM once per group, not
    // once per row tile (C5: 7.9 GB of X^T re-reads per launch otherwise).
    const unsigned num_n = (N + BN - 1) / BN, num_m = static_cast<unsigned>((batch + BM - 1) / BM);
    const unsigned pid = blockIdx.x, group = pid / (kGroup * num_n), first_m = group * kGroup;
    const unsigned gm = min(num_m - first_m, kGroup), in_group = pid % (kGroup * num_n);
    const int c0 = static_cast<int>(in_group / gm) * BN;
    const std::size_t b0 = static_cast<std::size_t>(first_m + in_group % gm) * BM;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = (warp / (BN / WN)) * WM, wn = (warp % (BN / WN)) * WN;
    const int nchunks = (K + BK - 1) / BK;

    // B: thread t copies the pair 2 (t % 16) of rows t / 16 + 16 i (ld_bt is
    // even and the rows 16-byte aligned; the zero padding beyond K is stored)
    auto load_b = [&](int chunk, int buf) {
        const int k = 2 * (tid % (BK / 2)), kk = chunk * BK + k;
        const int nk = min(2, max(0, K - kk));
#pragma unroll
        for (int i = 0; i < BN / (kThreads / (BK / 2)); ++i) {
            const int c = tid / (BK / 2) + i * (kThreads / (BK / 2));
            const int bytes = c0 + c < N ? 8 * nk : 0;
            cp_async16(Bs + buf * BN * LDS_ + c * LDS_ + k, bt + (bytes ? (c0 + c) * ld_bt + kk : 0), bytes);
        }
    };
    // A, fp64: 16-byte pairs when rows are aligned, else an 8-byte copy per element
    auto load_a64 = [&](int chunk, int buf) {
        if (vec16) {
            const int k = 2 * (tid % (BK / 2)), kk = chunk * BK + k;
            const int nk = min(2, max(0, K - kk));
#pragma unroll
            for (int i = 0; i < BM / (kThreads / (BK / 2)); ++i) {
                const int m = tid / (BK / 2) + i * (kThreads / (BK / 2));
                const int bytes = b0 + m < batch ? 8 * nk : 0;
                cp_async16(As + buf * BM * LDS_ + m * LDS_ + k,
                           reinterpret_cast<const double*>(in) + (bytes ? (b0 + m) * ld_in + kk : 0), bytes);
            }
            return;
        }
        const int k = tid % BK, kk = chunk * BK + k;
        const int src = kk < K ? (a_map ? __ldg(a_map + kk) : kk) : 0;
#pragma unroll
        for (int i = 0; i < BM / (kThreads / BK); ++i) {
            const int m = tid / BK + i * (kThreads / BK);
            const bool ok = kk < K && b0 + m < batch;
            cp_async8(As + buf * BM * LDS_ + m * LDS_ + k,
                      reinterpret_cast<const double*>(in) + (ok ? (b0 + m) * ld_in + src : 0), ok);
        }
    };
    // A, fp32: one chunk prefetched into registers, widened on the store
    constexpr int kAR = BM * BK / kThreads;
    float ra[kAR];
    auto fetch_a32 = [&](int chunk) {
        const int k = tid % BK, kk = chunk * BK + k;
        const int src = kk < K ? (a_map ? __ldg(a_map + kk) : kk) : 0;
#pragma unroll
        for (int i = 0; i < kAR; ++i) {
            const std::size_t b = b0 + tid / BK + i * (kThreads / BK);
            ra[i] = kk < K && b < batch ? reinterpret_cast<const float*>(in)[b * ld_in + src] : 0.f;
        }
    };
    auto store_a32 = [&](int buf) {
#pragma unroll
        for (int i = 0; i < kAR; ++i)
            As[buf * BM * LDS_ + (tid / BK + i * (kThreads / BK)) * LDS_ + tid % BK] = static_cast<double>(ra[i]);
    };
    constexpr bool F32 = sizeof(T) == 4;

    double acc[MF][NF][2];
#pragma unroll
    for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    load_b(0, 0);
    if constexpr (F32) {
        fetch_a32(0);
        store_a32(0);
    } else {
        load_a64(0, 0);
    }
    cp_async_commit();
    for (int ch = 0; ch < nchunks; ++ch) {
        const int buf = ch & 1;
        const bool more = ch + 1 < nchunks;
        if (more) {
            load_b(ch + 1, buf ^ 1);
            if constexpr (F32)
                fetch_a32(ch + 1);
            else
                load_a64(ch + 1, buf ^ 1);
        }
        cp_async_commit();
        cp_async_wait1();
        __syncthreads();
        const double* Ab = As + buf * BM * LDS_ + (wm + (lane >> 2)) * LDS_ + (lane & 3);
        const double* Bb = Bs + buf * BN * LDS_ + (wn + (lane >> 2)) * LDS_ + (lane & 3);
#pragma unroll
        for (int ks = 0; ks < BK / 4; ++ks) {
            double a[MF], bv[NF];
#pragma unroll
            for (int i = 0; i < MF; ++i) a[i] = Ab[i * 8 * LDS_ + ks * 4];
#pragma unroll
            for (int j = 0; j < NF; ++j) bv[j] = Bb[j * 8 * LDS_ + ks * 4];
#pragma unroll
            for (int i = 0; i < MF; ++i)
#pragma unroll
                for (int j = 0; j < NF; ++j) ptx::dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], bv[j]);
        }
        if constexpr (F32) {
            if (more) store_a32(buf ^ 1); // that buffer was last read before the previous barrier
        }
        __syncthreads();
    }

    bool bad = false;
#pragma unroll
    for (int i = 0; i < MF; ++i) {
        const std::size_t b = b0 + wm + i * 8 + (lane >> 2);
        if (b >= batch) continue;
        T* orow = out + b * ld_out;
#pragma unroll
        for (int j = 0; j < NF; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = c0 + wn + j * 8 + 2 * (lane & 3) + e;
                if (c < N) {
                    bad |= !isfinite(acc[i][j][e]);
                    if (fold_add) { // unfold: x_c = w_c + v_c, x_{2N-1-c} = w_c - v_c
                        const double w = static_cast<double>(fold_add[b * ld_add + c]);
                        orow[c] = static_cast<T>(w + acc[i][j][e]);
                        orow[2 * N - 1 - c] = static_cast<T>(w - acc[i][j][e]);
                    } else {
                        orow[col_map ? __ldg(col_map + c) : c] = static_cast<T>(acc[i][j][e]);
                    }
                }
            }
    }
    if (bad) atomicOr(flag, 1);
}

} // namespace

template <class T>
cudaError_t rows_by_basis(const T* in, std::size_t ld_in, const double* bt, std::size_t ld_bt, int K, int N, T* out,
                          std::size_t ld_out, std::size_t batch, int* flag, cudaStream_t stream, const int* col_map,
                          const int* a_map, const T* fold_add, std::size_t ld_add) {
    if (batch == 0 || N == 0) return cudaSuccess;
    if (ld_bt % 2 != 0 || reinterpret_cast<std::uintptr_t>(bt) % 16 != 0) return cudaErrorInvalidValue;
    constexpr std::size_t smem = 2 * (BM + BN) * LDS_ * sizeof(double);
    const cudaError_t attr = smem_optin(reinterpret_cast<const void*>(rows_by_basis_kernel<T>),
                                        static_cast<int>(smem));
    if (attr != cudaSuccess) return attr;
    const int vec16 = !a_map && (reinterpret_cast<std::uintptr_t>(in) % 16 == 0) && (ld_in % 2 == 0);
    const std::size_t num_n = (N + BN - 1) / BN;
    static const unsigned group = [] {
        const char* e = std::getenv("DCTP_TILE_GROUP");
        return e ? static_cast<unsigned>(std::max(1, std::atoi(e))) : 16u;
    }();
    const std::size_t kMaxRows = std::size_t{0x7fffffff} / num_n / BM * BM; // one-dimensional grid limit
    for (std::size_t r0 = 0; r0 < batch; r0 += kMaxRows) {
        const std::size_t rows = batch - r0 < kMaxRows ? batch - r0 : kMaxRows;
        const unsigned grid = static_cast<unsigned>(num_n * ((rows + BM - 1) / BM));
        rows_by_basis_kernel<T><<<grid, kThreads, smem, stream>>>(in + r0 * ld_in, ld_in, bt, ld_bt, K, N,
                                                                  out + r0 * ld_out, ld_out, rows, flag, vec16,
                                                                  col_map, a_map,
                                                                  fold_add ? fold_add + r0 * ld_add : nullptr, ld_add,
                                                                  group);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template cudaError_t rows_by_basis<double>(const double*, std::size_t, const double*, std::size_t, int, int, double*,
                                           std::size_t, std::size_t, int*, cudaStream_t, const int*, const int*,
                                           const double*, std::size_t);
template cudaError_t rows_by_basis<float>(const float*, std::size_t, const double*, std::size_t, int, int, float*,
                                          std::size_t, std::size_t, int*, cudaStream_t, const int*, const int*,
                                          const float*, std::size_t);

} // namespace dctp::dev

// --- materialising a plan's basis on the device -----------------------------------

namespace dctp::dev {
namespace {

/// Row s of the basis in the DCT domain, signed: sigma_s e_idx for a
/// pass-through slot, sigma_s a_s z_j / (lambda_j - nu_s) (z_j != 0) for an
/// active one (cauchy.hpp:90-98; the host's basis_coefficients, same ops).
__global__ void basis_coeff_kernel(int n, std::size_t ld, const double* __restrict__ z,
                                   const double* __restrict__ lambda, const double* __restrict__ nu,
                                   const int* __restrict__ pass_idx, const double* __restrict__ a,
                                   const double* __restrict__ sigma, double* __restrict__ y) {
    const int s = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int pidx = pass_idx[s];
    double v;
    if (pidx >= 0) {
        v = j == pidx ? 1.0 : 0.0;
    } else {
        const double zj = z[j];
        v = zj != 0.0 ? __ddiv_rn(__dmul_rn(a[s], zj), __dsub_rn(lambda[j], nu[s])) : 0.0;
    }
    y[static_cast<std::size_t>(s) * ld + j] = sigma[s] < 0.0 ? -v : v;
}

__global__ void transpose_kernel(const double* __restrict__ in, std::size_t ld_in, double* __restrict__ out,
                                 std::size_t ld_out, int n) {
    __shared__ double tile[32][33];
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int y = y0 + r, x = x0 + threadIdx.x;
        if (y < n && x < n) tile[r][threadIdx.x] = in[static_cast<std::size_t>(y) * ld_in + x];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int y = x0 + r, x = y0 + threadIdx.x;
        if (y < n && x < n) out[static_cast<std::size_t>(y) * ld_out + x] = tile[threadIdx.x][r];
    }
}

} // namespace

cudaError_t basis_coefficients(int n, std::size_t ld, const double* z, const double* lambda, const double* nu,
                               const int* pass_idx, const double* a, const double* sigma, double* y,
                               cudaStream_t stream, int rows) {
    if (n == 0) return cudaSuccess;
    if (rows < 0) rows = n;
    if (rows == 0) return cudaSuccess;
    dim3 grid(static_cast<unsigned>((n + 255) / 256), static_cast<unsigned>(rows));
    basis_coeff_kernel<<<grid, 256, 0, stream>>>(n, ld, z, lambda, nu, pass_idx, a, sigma, y);
    return cudaGetLastError();
}

cudaError_t transpose_square(const double* in, std::size_t ld_in, double* out, std::size_t ld_out, int n,
                             cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    dim3 grid(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((n + 31) / 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, stream>>>(in, ld_in, out, ld_out, n);
    return cudaGetLastError();
}

} // namespace dctp::dev
