// Fused persistent forward DCT+ for small plans (power-of-two n <= 512, at
// most 128 kept DCT indices and 128 secular roots), fp64, sm_100a.
//
// One CTA per SM loops over tiles of TS signals:
//   TMA 1-D bulk load of the tile (double-buffered, mbarrier completion)
//   -> orthonormal DCT-II of every row in shared memory: Makhoul packing fused
//      into the first Stockham pass of an n/2-point complex FFT (radix-2/4,
//      natural order), then the real split and e^{-i pi k/2n} rotation
//   -> each coefficient is routed once: kept indices into the A tile of the
//      Cauchy product, pass-through indices (signed) straight into their
//      output slot (fast_transform.hpp:171)
//   -> Cauchy stage on the fp64 tensor cores (mma.sync m8n8k4 DMMA):
//      out[s, slot_c] = sum_k shat[s, kept_k] * T[k, c] with
//      T[k, c] = sigma_c a_c z_k / (lambda_k - mu_c) (the reference's dense
//      T_r of fast_transform.hpp:355-366, transposed) held in REGISTERS as
//      m8n8k4 B fragments for the whole kernel (K x A <= 128 x 128 fp64 =
//      128 KB spread over 16 warps, one 8-column N-tile each)
//   -> the assembled output tile leaves with one TMA 1-D bulk store.
// HBM traffic is the algorithmic minimum (read s once, write the coefficients
// once); the Cauchy matrix is generated once per CTA from fp64 gaps.
#include <algorithm>

#include "kernels/common.cuh"
#include "kernels/launch.hpp"

namespace dctp::dev {
namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32; // one 8-slot N-tile of the Cauchy product per warp: A <= 128
constexpr int KTMAX = 32;            // k-tiles of 4: K <= 128
constexpr int LDA = KTMAX * 4 + 4;   // A-tile row stride (doubles): +4 staggers the 8 fragment rows over banks

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

template <int R>
__device__ __forceinline__ void butterfly(double2 (&v)[R]);

template <>
__device__ __forceinline__ void butterfly<2>(double2 (&v)[2]) {
    const double2 a = v[0], b = v[1];
    v[0] = make_double2(a.x + b.x, a.y + b.y);
    v[1] = make_double2(a.x - b.x, a.y - b.y);
}

template <>
__device__ __forceinline__ void butterfly<4>(double2 (&v)[4]) {
    // forward radix-4 DFT (e^{-2 pi i / 4} = -i)
    const double2 a0 = make_double2(v[0].x + v[2].x, v[0].y + v[2].y);
    const double2 a1 = make_double2(v[0].x - v[2].x, v[0].y - v[2].y);
    const double2 a2 = make_double2(v[1].x + v[3].x, v[1].y + v[3].y);
    const double2 a3 = make_double2(v[1].y - v[3].y, v[3].x - v[1].x); // -i (v1 - v3)
    v[0] = make_double2(a0.x + a2.x, a0.y + a2.y);
    v[2] = make_double2(a0.x - a2.x, a0.y - a2.y);
    v[1] = make_double2(a1.x + a3.x, a1.y + a3.y);
    v[3] = make_double2(a1.x - a3.x, a1.y - a3.y);
}

/// One Stockham (autosort) pass of radix R over TS rows of N points:
/// NS = size of the sub-transforms already done (log2 in lns).  FIRST: the
/// source is the real signal tile, packed on the fly (Makhoul:
/// w_m = v_{2m} + i v_{2m+1}, v = (x0, x2, ..., x3, x1)).
template <int N, int TS, int R, bool FIRST>
__device__ __forceinline__ void stockham_pass(const double2* __restrict__ src, const double* __restrict__ x,
                                              double2* __restrict__ dst, const double2* __restrict__ tw, int lns,
                                              int rows, bool& bad) {
    constexpr int M = N / R;
    constexpr int n = 2 * N;
    const int ns = 1 << lns;
    for (int t = threadIdx.x; t < TS * M; t += kThreads) {
        const int sig = t / M, j = t % M;
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int m = j + r * M;
            if constexpr (FIRST) {
                const double* xr = x + sig * n;
                const int p0 = 2 * m, p1 = 2 * m + 1;
                const double e0 = (p0 < N) ? xr[2 * p0] : xr[2 * (n - 1 - p0) + 1];
                const double e1 = (p1 < N) ? xr[2 * p1] : xr[2 * (n - 1 - p1) + 1];
                if (sig < rows) bad |= !isfinite(e0) || !isfinite(e1);
                v[r] = make_double2(e0, e1);
            } else {
                v[r] = src[sig * N + m];
            }
        }
        const int jm = j & (ns - 1);
        if (!FIRST || ns > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw[(r * jm * (N >> lns)) / R]);
        }
        butterfly<R>(v);
        const int d = ((j >> lns) << lns) * R + jm;
#pragma unroll
        for (int r = 0; r < R; ++r) dst[sig * N + d + r * ns] = v[r];
    }
}

/// The full n/2-point FFT of every row; returns the buffer holding the result.
template <int N, int TS>
__device__ __forceinline__ double2* fft_rows(const double* x, double2* a, double2* b, const double2* tw, int rows,
                                             bool& bad) {
    constexpr int LOGN = __builtin_ctz(N);
    int lns = 0;
    double2* src = nullptr;
    double2* dst = a;
    if constexpr (LOGN % 2 == 1) {
        stockham_pass<N, TS, 2, true>(nullptr, x, dst, tw, 0, rows, bad);
        lns = 1;
    } else {
        stockham_pass<N, TS, 4, true>(nullptr, x, dst, tw, 0, rows, bad);
        lns = 2;
    }
    __syncthreads();
    src = dst;
    dst = b;
#pragma unroll 1
    for (; lns < LOGN; lns += 2) {
        stockham_pass<N, TS, 4, false>(src, nullptr, dst, tw, lns, rows, bad);
        __syncthreads();
        double2* t = src;
        src = dst;
        dst = t;
    }
    return src;
}

template <int LOGN, int KT, int TS>
__global__ void __launch_bounds__(kThreads, 1)
fused_small_fwd_kernel(const double* __restrict__ in, double* __restrict__ out, std::size_t batch, SmallPlanDev P,
                       int* flag) {
    constexpr int n = 1 << LOGN, N = n / 2, MT = TS / 8;
    extern __shared__ __align__(128) unsigned char smem[];
    double* xbuf = reinterpret_cast<double*>(smem);
    double2* ca = reinterpret_cast<double2*>(xbuf + 2 * TS * n);
    double2* cb = ca + TS * N;
    double* atile = reinterpret_cast<double*>(cb + TS * N);
    double2* tw = reinterpret_cast<double2*>(atile + TS * LDA);
    double2* sp = tw + N;
    double2* rt = sp + N;
    int* route = reinterpret_cast<int*>(rt + N + 1);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(route + n);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < N; i += kThreads) {
        tw[i] = reinterpret_cast<const double2*>(P.fft_tw)[i];
        sp[i] = reinterpret_cast<const double2*>(P.split_tw)[i];
    }
    for (int i = tid; i <= N; i += kThreads) rt[i] = reinterpret_cast<const double2*>(P.rot_tw)[i];
    for (int i = tid; i < n; i += kThreads) route[i] = P.route[i];
    for (int i = tid; i < TS * LDA; i += kThreads) atile[i] = 0.0;
    if (tid == 0) {
        ptx::mbar_init(&mbar[0], 1);
        ptx::mbar_init(&mbar[1], 1);
        ptx::fence_mbar_init();
    }

    // Cauchy fragments, resident for the whole kernel: B[k][c] = T[k][c] for
    // this warp's 8 output columns c and all K (zero-padded to 4*KT) kept rows.
    double bf[KT];
    {
        const int c = warp * 8 + (lane >> 2);
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
            const int k = kt * 4 + (lane & 3);
            double v = 0.0;
            if (k < P.K && c < P.A) v = P.act_scale[c] * (P.z_kept[k] / (P.lam_kept[k] - P.nu[c]));
            bf[kt] = v;
        }
    }
    int slot[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int c = warp * 8 + 2 * (lane & 3) + e;
        slot[e] = c < P.A ? P.act_slot[c] : -1;
    }
    __syncthreads();

    const std::size_t ntiles = (batch + TS - 1) / TS;
    auto issue = [&](std::size_t tile, int b) {
        const std::size_t rows = min(static_cast<std::size_t>(TS), batch - tile * TS);
        const uint32_t bytes = static_cast<uint32_t>(rows * n * sizeof(double));
        ptx::mbar_expect_tx(&mbar[b], bytes);
        ptx::bulk_load(xbuf + b * TS * n, in + tile * TS * n, bytes, &mbar[b]);
    };
    if (tid == 0) {
        if (blockIdx.x < ntiles) issue(blockIdx.x, 0);
        if (blockIdx.x + gridDim.x < ntiles) issue(blockIdx.x + gridDim.x, 1);
    }

    const double scale = sqrt(2.0 / n);
    const double dc_scale = 1.0 / sqrt(static_cast<double>(n));
    bool bad = false;
    int it = 0;
    for (std::size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int b = it & 1;
        double* x = xbuf + b * TS * n;
        const int rows = static_cast<int>(min(static_cast<std::size_t>(TS), batch - tile * TS));
        ptx::mbar_wait(&mbar[b], (it >> 1) & 1);

        const double2* F = fft_rows<N, TS>(x, ca, cb, tw, rows, bad);

        // split + rotate + scale, then route every coefficient once
        auto put = [&](int r, int j, double v) {
            const int d = route[j];
            if (d >= 0) {
                atile[r * LDA + d] = v;
            } else {
                const int p = -d - 1;
                x[r * n + (p >> 1)] = (p & 1) ? -v : v;
            }
        };
        for (int t = tid; t < TS * N; t += kThreads) {
            const int r = t / N, k = t % N;
            const double2* row = F + r * N;
            if (k == 0) {
                const double2 w0 = row[0];
                put(r, 0, (w0.x + w0.y) * dc_scale);
                put(r, N, (w0.x - w0.y) * rt[N].x * scale);
                continue;
            }
            const double2 wk = row[k], wc = row[N - k];
            const double er = 0.5 * (wk.x + wc.x), ei = 0.5 * (wk.y - wc.y);
            const double orr = 0.5 * (wk.x - wc.x), oi = 0.5 * (wk.y + wc.y);
            const double2 s2 = sp[k];
            const double qr = s2.x * orr - s2.y * oi, qi = s2.x * oi + s2.y * orr;
            const double vr = er + qi, vi = ei - qr;
            const double2 c2 = rt[k];
            put(r, k, (vr * c2.x - vi * c2.y) * scale);
            put(r, n - k, -(vr * c2.y + vi * c2.x) * scale);
        }
        __syncthreads();

        // Cauchy stage: D[s, c] += A[s, k] * B[k, c] on DMMA, 8 x 8 x 4 at a time.
        double acc[MT][2];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
        const double* arow = atile + (lane >> 2) * LDA + (lane & 3);
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
            double a[MT];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) a[mt] = arow[mt * 8 * LDA + kt * 4];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) ptx::dmma_8x8x4(acc[mt][0], acc[mt][1], a[mt], bf[kt]);
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const int r = mt * 8 + (lane >> 2);
#pragma unroll
            for (int e = 0; e < 2; ++e)
                if (slot[e] >= 0) x[r * n + slot[e]] = acc[mt][e];
        }
        ptx::fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            ptx::bulk_store(out + tile * TS * n, x, static_cast<uint32_t>(rows * n * sizeof(double)));
            ptx::bulk_commit();
            const std::size_t next = tile + 2 * static_cast<std::size_t>(gridDim.x);
            if (next < ntiles) {
                ptx::bulk_wait_read_all();
                issue(next, b);
            }
        }
    }
    if (bad) atomicOr(flag, 1);
    if (tid == 0) ptx::bulk_wait_all();
}

template <int LOGN, int TS>
constexpr std::size_t smem_bytes() {
    constexpr int n = 1 << LOGN, N = n / 2;
    return 2 * TS * n * sizeof(double) + 2 * TS * N * sizeof(double2) + TS * LDA * sizeof(double) +
           (3 * N + 1) * sizeof(double2) + n * sizeof(int) + 2 * sizeof(uint64_t);
}

template <int LOGN, int KT>
cudaError_t launch_small(const double* in, double* out, std::size_t batch, const SmallPlanDev& P, int* flag,
                         int num_sms, cudaStream_t stream) {
    constexpr int TS = LOGN >= 9 ? 8 : 16;
    constexpr std::size_t smem = smem_bytes<LOGN, TS>();
    auto kern = fused_small_fwd_kernel<LOGN, KT, TS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const std::size_t ntiles = (batch + TS - 1) / TS;
    const unsigned grid = static_cast<unsigned>(std::min<std::size_t>(ntiles, static_cast<std::size_t>(num_sms)));
    kern<<<grid, kThreads, smem, stream>>>(in, out, batch, P, flag);
    return cudaGetLastError();
}

/// K is padded up to 4*KT with KT in {4, 8, 16, 32} (never above n/4).
template <int LOGN>
cudaError_t dispatch_kt(const double* in, double* out, std::size_t batch, const SmallPlanDev& P, int* flag,
                        int num_sms, cudaStream_t stream) {
    constexpr int n = 1 << LOGN;
    if (P.K <= 16 || n <= 16) return launch_small<LOGN, 4>(in, out, batch, P, flag, num_sms, stream);
    if constexpr (n >= 32)
        if (P.K <= 32 || n <= 32) return launch_small<LOGN, 8>(in, out, batch, P, flag, num_sms, stream);
    if constexpr (n >= 64)
        if (P.K <= 64 || n <= 64) return launch_small<LOGN, 16>(in, out, batch, P, flag, num_sms, stream);
    if constexpr (n >= 128) return launch_small<LOGN, 32>(in, out, batch, P, flag, num_sms, stream);
    return cudaErrorInvalidValue;
}

} // namespace

bool fused_small_supported(std::size_t n, int K, int A) {
    return is_pow2(n) && n >= 16 && n <= 512 && K <= 4 * KTMAX && A <= 8 * kWarps;
}

cudaError_t fused_small_forward(const double* in, double* out, std::size_t batch, const SmallPlanDev& P, int* flag,
                                int num_sms, cudaStream_t stream) {
    if (batch == 0) return cudaSuccess;
    switch (P.n) {
        case 16: return dispatch_kt<4>(in, out, batch, P, flag, num_sms, stream);
        case 32: return dispatch_kt<5>(in, out, batch, P, flag, num_sms, stream);
        case 64: return dispatch_kt<6>(in, out, batch, P, flag, num_sms, stream);
        case 128: return dispatch_kt<7>(in, out, batch, P, flag, num_sms, stream);
        case 256: return dispatch_kt<8>(in, out, batch, P, flag, num_sms, stream);
        case 512: return dispatch_kt<9>(in, out, batch, P, flag, num_sms, stream);
        default: return cudaErrorInvalidValue;
    }
}

} // namespace dctp::dev
