// Cauchy stage of DCT+ on the fp64 tensor cores (DMMA), for plans too large
// for the fused kernel (C3: 512 x 512, C5: 8192 x 8192, progressive members):
//
//   out[b, dst[c]] = cscale[c] * sum_r in[b, src[r]] * rscale[r] / (x[r] - y[c])
//
// A dense GEMM [batch x R] x [R x C] whose B operand is never stored: each CTA
// generates its 32 x 128 B chunk in shared memory from fp64 gaps
// right before using it, so HBM traffic is only the signal
// rows in and the coefficients out (C5's materialised T would be 512 MB and
// would be re-read once per row tile).  A rows are gathered with cp.async
// (LDGSTS, 8-byte elements) one chunk ahead.  CTA tile 64 x 128 (two CTAs per
// SM; a 128-row tile left C3's 512 CTAs at 3.5 waves), 8 warps of 32 x 32,
// m8n8k4 DMMA fragments loaded from rows padded to 36 doubles.  The division
// per generated entry is amortised over 64 signals.  (m16n8k16 fragments,
// tools/mma16_layout.cu, issue 8x fewer DMMA instructions but measured no
// faster: the kernel is not issue-bound.)
#include <algorithm>
#include <cstdint>

#include "kernels/common.cuh"
#include "kernels/launch.hpp"

namespace dctp::dev {
namespace {

constexpr int BM = 64, BN = 128, BK = 32, LDS_ = BK + 4;
constexpr int kThreads = 256;
constexpr int WM = 32, WN = 32;         // warp tile
constexpr int MF = WM / 8, NF = WN / 8; // fragments per warp

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
    const unsigned s = ptx::smem_addr(smem);
    const int bytes = pred ? 8 : 0; // zero-fill when out of range
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(kThreads, 2)
cauchy_dmma_kernel(const double* __restrict__ in, std::size_t ld_in, double* __restrict__ out, std::size_t ld_out,
                   const CauchyStage* __restrict__ stages, std::size_t batch, int* flag, int vec16) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* As = reinterpret_cast<double*>(smem_raw); // 2 x BM x LDS_
    double* Bs = As + 2 * BM * LDS_;                  // 2 x BN x LDS_ (transposed: [c][k])
    double* ys = Bs + 2 * BN * LDS_;                  // BN: the tile's column nodes y_c
    const CauchyStage st = stages[blockIdx.z];
    const int c0 = blockIdx.x * BN; // column tiles fastest: CTAs sharing a row tile run together (A from L2)
    if (c0 >= st.cols) return;
    const std::size_t b0 = static_cast<std::size_t>(blockIdx.y) * BM;
    const double* rscale = static_cast<const double*>(st.rscale);
    const double* cscale = static_cast<const double*>(st.cscale);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = (warp / (BN / WN)) * WM, wn = (warp % (BN / WN)) * WN;
    const int nchunks = (st.rows + BK - 1) / BK;
    for (int c = tid; c < BN; c += kThreads) ys[c] = c0 + c < st.cols ? st.y[c0 + c] : 0.0;
    __syncthreads();

    // A rows: compacted inputs (src_contig) load as 16-byte pairs, otherwise an
    // 8-byte gather through src[].  Thread t copies column k = t % 32 (or the
    // pair 2 (t % 16)) of rows t / 32 + 8 i (or t / 16 + 16 i).
    auto load_a = [&](int chunk, int buf) {
        if (st.src_contig && vec16) {
            const int k = 2 * (tid % (BK / 2)), r = chunk * BK + k;
            const int nk = min(2, max(0, st.rows - r)); // valid elements of the pair
#pragma unroll
            for (int i = 0; i < BM / (kThreads / (BK / 2)); ++i) {
                const int m = tid / (BK / 2) + i * (kThreads / (BK / 2));
                const std::size_t b = b0 + m;
                const int bytes = b < batch ? 8 * nk : 0;
                const unsigned sa = ptx::smem_addr(As + buf * BM * LDS_ + m * LDS_ + k);
                const double* ga = in + (bytes ? b * ld_in + r : 0);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(ga), "r"(bytes)
                             : "memory");
            }
            return;
        }
        const int k = tid % BK, r = chunk * BK + k;
        const bool kin = r < st.rows;
        const int src = kin ? st.src[r] : 0;
#pragma unroll
        for (int i = 0; i < BM / (kThreads / BK); ++i) {
            const int m = tid / BK + i * (kThreads / BK);
            const std::size_t b = b0 + m;
            const bool ok = kin && b < batch;
            cp_async8(As + buf * BM * LDS_ + m * LDS_ + k, in + (ok ? b * ld_in + src : 0), ok);
        }
    };
    // B generation: lane = k within the chunk (one contiguous 256-byte row store
    // per column, conflict-free), warp w fills columns w, w + 8, ..., w + 120.
    // x and rscale of the chunk's rows are fetched one chunk ahead (their L2
    // latency would otherwise stall every chunk's B generation)
    auto fetch_xr = [&](int chunk, double& xr, double& sr) {
        const int r = chunk * BK + lane;
        xr = r < st.rows ? st.x[r] : 0.0;
        sr = r < st.rows ? rscale[r] : 0.0;
    };
    double xr_next = 0.0, sr_next = 0.0;
    fetch_xr(0, xr_next, sr_next);
    auto gen_b = [&](int chunk, int buf) {
        const int r = chunk * BK + lane;
        const bool rok = r < st.rows;
        const double xr = xr_next, sr = sr_next;
        if (chunk + 1 < nchunks) fetch_xr(chunk + 1, xr_next, sr_next);
        double* col = Bs + buf * BN * LDS_ + lane;
#pragma unroll 4
        for (int cc = warp; cc < BN; cc += kThreads / 32) {
            const int c = c0 + cc;
            double v = 0.0;
            if (rok && c < st.cols) { // padded rows stay exactly 0 (x = y would give 0 * inf)
                // rscale / (x - y): reciprocal by MUFU seed + two Newton steps (< 1 ulp)
                const double d = xr - ys[cc];
                double rcp;
                asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rcp) : "d"(d));
                double e = fma(-d, rcp, 1.0);
                rcp = fma(rcp, e, rcp);
                e = fma(-d, rcp, 1.0);
                rcp = fma(rcp, e, rcp);
                v = sr * rcp;
            }
            col[cc * LDS_] = v;
        }
    };

    double acc[MF][NF][2];
#pragma unroll
    for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    load_a(0, 0);
    cp_async_commit();
    for (int ch = 0; ch < nchunks; ++ch) {
        const int buf = ch & 1;
        if (ch + 1 < nchunks) load_a(ch + 1, buf ^ 1);
        cp_async_commit();
        gen_b(ch, buf);
        cp_async_wait<1>();
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
        __syncthreads();
    }

    // epilogue: out[b, dst[c]] = cscale[c] * acc; non-finite inputs show up here
    bool bad = false;
#pragma unroll
    for (int i = 0; i < MF; ++i) {
        const std::size_t b = b0 + wm + i * 8 + (lane >> 2);
        if (b >= batch) continue;
        double* orow = out + b * ld_out + st.out_offset;
#pragma unroll
        for (int j = 0; j < NF; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = c0 + wn + j * 8 + 2 * (lane & 3) + e;
                if (c < st.cols) {
                    const double v = cscale[c] * acc[i][j][e];
                    bad |= !isfinite(v);
                    orow[st.dst[c]] = v;
                }
            }
    }
    if (bad) atomicOr(flag, 1);
}

} // namespace

cudaError_t cauchy_rows_dmma(const double* in, std::size_t ld_in, double* out, std::size_t ld_out,
                             const CauchyStage* stages_dev, int num_stages, int max_cols, std::size_t batch,
                             int* flag, cudaStream_t stream) {
    if (batch == 0 || num_stages == 0 || max_cols == 0) return cudaSuccess;
    constexpr std::size_t smem = 2 * (BM + BN) * LDS_ * sizeof(double) + BN * sizeof(double);
    const cudaError_t attr = smem_optin(reinterpret_cast<const void*>(cauchy_dmma_kernel), static_cast<int>(smem));
    if (attr != cudaSuccess) return attr;
    // 16-byte row loads need 16-byte aligned rows (otherwise the 8-byte gather runs)
    const int vec16 = (reinterpret_cast<std::uintptr_t>(in) % 16 == 0) && (ld_in % 2 == 0);
    constexpr std::size_t kMaxRows = std::size_t{65535} * BM; // gridDim.y limit
    for (std::size_t r0 = 0; r0 < batch; r0 += kMaxRows) {
        const std::size_t rows = batch - r0 < kMaxRows ? batch - r0 : kMaxRows;
        dim3 grid(static_cast<unsigned>((max_cols + BN - 1) / BN), static_cast<unsigned>((rows + BM - 1) / BM),
                  static_cast<unsigned>(num_stages));
        cauchy_dmma_kernel<<<grid, kThreads, smem, stream>>>(in + r0 * ld_in, ld_in, out + r0 * ld_out, ld_out,
                                                             stages_dev, rows, flag, vec16);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

} // namespace dctp::dev
