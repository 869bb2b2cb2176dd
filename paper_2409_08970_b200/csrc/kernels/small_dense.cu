// Latency kernel for small plans (n <= 128) and small batches, sm_100a:
//
//   out[b, c] = sum_k in[b, k] * xt[c, k]            (xt = X^T, the plan's basis)
//
// one launch, one CTA per 32 signals: the CTA copies X^T (n x n fp64, L2
// resident after the first CTA) and its 32 rows into shared memory with
// 16-byte loads, then 8 warps run m8n8k4 DMMA over 8 x 8 output blocks and
// store.  No pipeline, no persistent scheduling, no TMA: for C1 (4096
// signals of n = 64) the fused persistent kernel spends most of its 15 us in
// per-CTA setup (T in registers, twiddles, barrier ring) for ~1 us of
// arithmetic; this kernel's critical path is one L2 round trip plus 64 DMMAs
// per warp.  The dense product is exact math (the basis X from the plan's
// setup), the same route forward_nmvp takes (fast_transform.hpp:199-209).
#include <cstdint>

#include "kernels/common.cuh"
#include "kernels/launch.hpp"

namespace dctp::dev {
namespace {

constexpr int SIG = 32;   // signals per CTA
constexpr int kThreads = 256;

template <int N>
__global__ void __launch_bounds__(kThreads)
small_dense_kernel(const double* __restrict__ in, std::size_t ld_in, const double* __restrict__ xt, std::size_t ld_xt,
                   double* __restrict__ out, std::size_t ld_out, std::size_t batch, int* flag) {
    constexpr int LD = N + 2;          // padded rows (doubles)
    extern __shared__ __align__(16) double sm[];
    double* xs = sm;                    // N x LD (X^T rows)
    double* ss = sm + N * LD;           // SIG x LD (signals)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const std::size_t b0 = static_cast<std::size_t>(blockIdx.x) * SIG;
    // X^T and the signal rows into shared memory, 16 bytes per load
    for (int i = tid; i < N * (N / 2); i += kThreads) {
        const int r = i / (N / 2), c = 2 * (i % (N / 2));
        const double2 v = __ldg(reinterpret_cast<const double2*>(xt + static_cast<std::size_t>(r) * ld_xt + c));
        xs[r * LD + c] = v.x;
        xs[r * LD + c + 1] = v.y;
    }
    bool bad = false;
    for (int i = tid; i < SIG * (N / 2); i += kThreads) {
        const int r = i / (N / 2), c = 2 * (i % (N / 2));
        double2 v = make_double2(0.0, 0.0);
        if (b0 + r < batch) v = __ldg(reinterpret_cast<const double2*>(in + (b0 + r) * ld_in + c));
        bad |= !isfinite(v.x) || !isfinite(v.y);
        ss[r * LD + c] = v.x;
        ss[r * LD + c + 1] = v.y;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
    __syncthreads();
    // output blocks: (SIG / 8) signal blocks x (N / 8) column blocks over 8 warps
    constexpr int SB = SIG / 8, CB = N / 8, PER = SB * CB / 8;
    double acc[PER][2];
#pragma unroll
    for (int p = 0; p < PER; ++p) acc[p][0] = acc[p][1] = 0.0;
    const int ar = lane >> 2, ak = lane & 3;
#pragma unroll 4
    for (int k0 = 0; k0 < N; k0 += 4) {
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            const int blk = warp * PER + p, sb = blk % SB, cb = blk / SB;
            const double a = ss[(sb * 8 + ar) * LD + k0 + ak];
            const double b = xs[(cb * 8 + ar) * LD + k0 + ak];
            ptx::dmma_8x8x4(acc[p][0], acc[p][1], a, b);
        }
    }
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

template <int N>
cudaError_t launch(const double* in, std::size_t ld_in, const double* xt, std::size_t ld_xt, double* out,
                   std::size_t ld_out, std::size_t batch, int* flag, cudaStream_t stream) {
    constexpr int smem = (N + SIG) * (N + 2) * static_cast<int>(sizeof(double));
    const cudaError_t e = smem_optin(reinterpret_cast<const void*>(small_dense_kernel<N>), smem);
    if (e != cudaSuccess) return e;
    const std::size_t grid = (batch + SIG - 1) / SIG;
    if (grid >= (1ull << 31)) return cudaErrorInvalidValue;
    small_dense_kernel<N><<<static_cast<unsigned>(grid), kThreads, smem, stream>>>(in, ld_in, xt, ld_xt, out, ld_out,
                                                                                  batch, flag);
    return cudaGetLastError();
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
