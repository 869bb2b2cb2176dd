// Latency kernel for small plans (n <= 128) and small batches, sm_100a:
//
//   out[b, c] = sum_k in[b, k] * xt[c, k]            (xt = X^T, the plan's basis)
//
// one launch, one CTA per 32 signals: the CTA copies X^T (n x n fp64, L2
// resident after the first CTA) and its rows into shared memory with 16-byte
// cp.async copies — all in flight at once, in two commit groups along k so
// the first half's products overlap the second half's copies — then 8 warps
// run m8n8k4 DMMA over 8 x 8 output blocks and store.  No pipeline, no persistent scheduling: for C1 (4096 signals of n =
// 64) the fused persistent kernel spends most of its 15 us in per-CTA setup
// (T in registers, twiddles, barrier ring) for ~1 us of arithmetic; this
// kernel's critical path is one memory round trip plus 16 DMMA steps per
// warp.  The dense product is exact math (the basis X from the plan's
// setup), the same route forward_nmvp takes (fast_transform.hpp:199-209).
#include <cstdint>
#include <cstdlib>

#include "kernels/common.cuh"
#include "kernels/launch.hpp"

namespace dctp::dev {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(ptx::smem_addr(smem)), "l"(gmem) : "memory");
}

template <int N, int SIG>
__global__ void __launch_bounds__(kThreads)
small_dense_kernel(const double* __restrict__ in, std::size_t ld_in, const double* __restrict__ xt, std::size_t ld_xt,
                   double* __restrict__ out, std::size_t ld_out, std::size_t batch, int* flag) {
    constexpr int LD = N + 2;          // padded rows (doubles; 16-byte aligned rows)
    extern __shared__ __align__(16) double sm[];
    double* xs = sm;                    // N x LD (X^T rows)
    double* ss = sm + N * LD;           // SIG x LD (signals)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const std::size_t b0 = static_cast<std::size_t>(blockIdx.x) * SIG;
    // X^T and the signal rows into shared memory, 16-byte cp.async copies, in
    // two commit groups along k: the first half's products start while the
    // second half's copies are still in flight
    constexpr int H = N / 4; // 16-byte copies per row half
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        for (int i = tid; i < N * H; i += kThreads) {
            const int r = i / H, c = 2 * (g * H + i % H);
            cp_async16(xs + r * LD + c, xt + static_cast<std::size_t>(r) * ld_xt + c);
        }
        for (int i = tid; i < SIG * H; i += kThreads) {
            const int r = i / H, c = 2 * (g * H + i % H);
            if (b0 + r < batch)
                cp_async16(ss + r * LD + c, in + (b0 + r) * ld_in + c);
            else
                *reinterpret_cast<double2*>(ss + r * LD + c) = make_double2(0.0, 0.0);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    // output blocks: (SIG / 8) signal blocks x (N / 8) column blocks over 8 warps
    constexpr int SB = SIG / 8, CB = N / 8, PER = SB * CB / 8;
    static_assert(PER >= 1 && SB * CB % 8 == 0, "8 warps x PER blocks of 8 x 8");
    double acc[PER][2];
#pragma unroll
    for (int p = 0; p < PER; ++p) acc[p][0] = acc[p][1] = 0.0;
    const int ar = lane >> 2, ak = lane & 3;
    bool bad = false; // check_signal: each thread reads back the signal words it copied
#pragma unroll 1
    for (int g = 0; g < 2; ++g) {
        if (g == 0)
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        else
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        for (int i = tid; i < SIG * H; i += kThreads) {
            const int r = i / H, c = 2 * (g * H + i % H);
            const double2 v = *reinterpret_cast<const double2*>(ss + r * LD + c);
            bad |= !isfinite(v.x) || !isfinite(v.y);
        }
        __syncthreads();
#pragma unroll 4
        for (int k0 = g * (N / 2); k0 < (g + 1) * (N / 2); k0 += 4) {
#pragma unroll
            for (int p = 0; p < PER; ++p) {
                const int blk = warp * PER + p, sb = blk % SB, cb = blk / SB;
                const double a = ss[(sb * 8 + ar) * LD + k0 + ak];
                const double b = xs[(cb * 8 + ar) * LD + k0 + ak];
                ptx::dmma_8x8x4(acc[p][0], acc[p][1], a, b);
            }
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
#pragma unroll
    for (int p = 0; p < PER; ++p) {
        const int blk = warp * PER + p, sb = blk % SB, cb = blk / SB;
        const std::size_t row = b0 + sb * 8 + ar;
        if (row < batch) {
            double* o = out + row * ld_out + cb * 8 + 2 * ak;
            *reinterpret_cast<double2*>(o) = make_double2(acc[p][0], acc[p][1]);
        }
    }
}

template <int N, int SIG>
cudaError_t launch_sig(const double* in, std::size_t ld_in, const double* xt, std::size_t ld_xt, double* out,
                       std::size_t ld_out, std::size_t batch, int* flag, cudaStream_t stream) {
    constexpr int smem = (N + SIG) * (N + 2) * static_cast<int>(sizeof(double));
    const cudaError_t e = smem_optin(reinterpret_cast<const void*>(small_dense_kernel<N, SIG>), smem);
    if (e != cudaSuccess) return e;
    const std::size_t grid = (batch + SIG - 1) / SIG;
    if (grid >= (1ull << 31)) return cudaErrorInvalidValue;
    small_dense_kernel<N, SIG><<<static_cast<unsigned>(grid), kThreads, smem, stream>>>(in, ld_in, xt, ld_xt, out,
                                                                                       ld_out, batch, flag);
    return cudaGetLastError();
}

/// 32 signals per CTA (DCTP_SMALL_DENSE_SIG = 16: 16 per CTA, more CTAs).
template <int N>
cudaError_t launch(const double* in, std::size_t ld_in, const double* xt, std::size_t ld_xt, double* out,
                   std::size_t ld_out, std::size_t batch, int* flag, cudaStream_t stream) {
    static const int forced = [] {
        const char* e = std::getenv("DCTP_SMALL_DENSE_SIG");
        return e ? std::atoi(e) : 0;
    }();
    const bool sig16 = forced == 16; // measured: 16 per CTA is slower even at C1's 128 CTAs (5.5 vs 5.2 us)
    if constexpr (N >= 32) // 16 signals x N / 8 column blocks: at least one 8 x 8 block per warp
        if (sig16) return launch_sig<N, 16>(in, ld_in, xt, ld_xt, out, ld_out, batch, flag, stream);
    return launch_sig<N, 32>(in, ld_in, xt, ld_xt, out, ld_out, batch, flag, stream);
}

} // namespace

bool small_dense_supported(std::size_t n, const void* in, std::size_t ld_in, const void* out, std::size_t ld_out) {
    const bool al = reinterpret_cast<std::uintptr_t>(in) % 16 == 0 && reinterpret_cast<std::uintptr_t>(out) % 16 == 0 &&
                    ld_in % 2 == 0 && ld_out % 2 == 0;
    return al && (n == 16 || n == 32 || n == 64 || n == 128);
}

cudaError_t small_dense_forward(const double* in, std::size_t ld_in, const double* xt, std::size_t ld_xt, double* out,
                                std::size_t ld_out, std::size_t n, std::size_t batch, int* flag, cudaStream_t stream) {
    if (batch == 0) return cudaSuccess;
    switch (n) {
        case 16: return launch<16>(in, ld_in, xt, ld_xt, out, ld_out, batch, flag, stream);
        case 32: return launch<32>(in, ld_in, xt, ld_xt, out, ld_out, batch, flag, stream);
        case 64: return launch<64>(in, ld_in, xt, ld_xt, out, ld_out, batch, flag, stream);
        case 128: return launch<128>(in, ld_in, xt, ld_xt, out, ld_out, batch, flag, stream);
        default: return cudaErrorInvalidValue;
    }
}

} // namespace dctp::dev
