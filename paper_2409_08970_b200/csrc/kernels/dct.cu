// Batched orthonormal DCT-II / DCT-III (the U^T s and U d stages of DCT+),
// sm_100a.  Replaces the reference's per-signal FFTW REDFT10/REDFT01 calls
// (proj/include/dctplus/trig.hpp:95-110) for a whole batch per launch.
//
// Power-of-two n: Makhoul's reordering turns the length-n DCT into one
// length-n/2 complex FFT of the packed real sequence, run in shared memory
// (bit-reversed load, radix-8 DIT passes, one CTA processes rows_per_cta signals
// at once), followed by the real-split and the e^{-i pi k/2n} rotation.  The
// epilogue stages the coefficients in shared memory and writes them with
// coalesced row stores plus an optional scattered "emit" list (pass-through
// slots of the DCT+ output), so the pass-through never needs its own launch.
// Other n: a direct O(n^2) kernel over a cos(pi m / 2n) table.
#include <algorithm>

#include <cuda_bf16.h>
#include <cmath>

#include "kernels/common.cuh"
#include "kernels/fft_smem.cuh"
#include "kernels/launch.hpp"

namespace dctp::dev {
namespace {

constexpr int kThreads = 256;
constexpr int kTileElems = 2048; // signal samples staged per CTA

/// Shared memory of the FFT kernels: natural buffer (later the real output
/// rows), working buffer; both rows_per_cta x padded_len(n/2) complex.
template <class T>
std::size_t fft_smem_bytes(std::size_t n, int rows) {
    return 2 * static_cast<std::size_t>(rows) * padded_len(static_cast<int>(n / 2)) * sizeof(T) * 2;
}

/// Byte offset of (row r, 16-byte chunk c16) in a K-major SWIZZLE_64B tile
/// row of 64 bytes — the int8 GEMM's operand image (ozaki.cu).
__device__ __forceinline__ uint32_t sw64_int8(int r, int c16) {
    return static_cast<uint32_t>(r * 64 + ((c16 ^ ((r >> 1) & 3)) << 4));
}

/// Four consecutive values at a 16-byte aligned address (float4 / 2 x double2).
__device__ __forceinline__ void load4(const float* p, float (&v)[4]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
}
__device__ __forceinline__ void load4(const double* p, double (&v)[4]) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p + 2));
    v[0] = a.x, v[1] = a.y, v[2] = b.x, v[3] = b.y;
}
__device__ __forceinline__ void store4(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void store4(double* p, const double (&v)[4]) {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    *reinterpret_cast<double2*>(p + 2) = make_double2(v[2], v[3]);
}

/// (t / K, t % K) for a thread's flat index t advanced by `step`, without a
/// division per element (the gather loops' index math was ~30% of their
/// instructions).
__device__ __forceinline__ void step_rk(int& r, int& k, int step, int K) {
    k += step;
    while (k >= K) {
        k -= K;
        ++r;
    }
}

/// Byte offset of (row grow, column k) in the int8 slice image of slice 0
/// (tiles of fs.tile_rows rows, 64-byte K chunks, SWIZZLE_64B), shifts for the
/// 128-row tiles every caller uses.
__device__ __forceinline__ std::size_t slice_off(const FoldSlices& fs, std::size_t grow, int k) {
    std::size_t tile;
    int lr;
    if (fs.tile_rows == 128) {
        tile = grow >> 7;
        lr = static_cast<int>(grow & 127);
    } else {
        tile = grow / fs.tile_rows;
        lr = static_cast<int>(grow % fs.tile_rows);
    }
    const std::size_t slice_bytes = static_cast<std::size_t>(fs.tile_rows) * 64;
    return ((tile * fs.nch + (k >> 6)) * fs.S) * slice_bytes + sw64_int8(lr, (k & 63) >> 4) + (k & 15);
}

/// Eight consecutive values k0..k0+7 of one row (src: the row, 16-byte
/// aligned when vec) scaled and cut into S int8 digits (ozaki_digit), one
/// 8-byte store per slice plane.
template <int S>
__device__ __forceinline__ void slice8_rows(const double* src, int k0, int K, bool vec, double scale, int8_t* dst,
                                            std::size_t slice_bytes) {
    double v[8];
    if (vec && k0 + 8 <= K) {
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
            const double2 p = *reinterpret_cast<const double2*>(src + k0 + u);
            v[u] = p.x;
            v[u + 1] = p.y;
        }
    } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = k0 + u < K ? src[k0 + u] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = isfinite(v[u]) ? v[u] * scale : 0.0;
#pragma unroll
    for (int sl = 0; sl < S; ++sl) {
        uint32_t lo = 0u, hi = 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            lo |= ozaki_digit(v[u]) << (8 * u);
            hi |= ozaki_digit(v[4 + u]) << (8 * u);
        }
        *reinterpret_cast<uint2*>(dst + sl * slice_bytes) = make_uint2(lo, hi);
    }
}

/// The slices of `rows` rows of K values each (src row r at src + r * lds),
/// 8-value groups spread over the CTA.
__device__ __forceinline__ void slice_rows(const double* src, int lds, int rows, int K, std::size_t b0,
                                           const FoldSlices& fs, const double* rscale) {
    const int groups = fs.nch * 8; // 8-value groups per row (64-byte chunks)
    const std::size_t slice_bytes = static_cast<std::size_t>(fs.tile_rows) * 64;
    const bool vec = (lds % 2) == 0;
    int r = threadIdx.x / groups, kg = threadIdx.x - r * groups;
    for (; r < rows; step_rk(r, kg, kThreads, groups)) {
        const int k0 = 8 * kg;
        int8_t* dst = fs.sl + slice_off(fs, b0 + r, k0);
        if (fs.S == 5)
            slice8_rows<5>(src + r * lds, k0, K, vec, rscale[r], dst, slice_bytes);
        else
            slice8_rows<6>(src + r * lds, k0, K, vec, rscale[r], dst, slice_bytes);
    }
}

__device__ __forceinline__ uint32_t bf16_pair(float a, float b) {
    return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(a))) |
           (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(b))) << 16);
}

/// fp32 rows (row r at src + r * lds, K values) -> the bf16x3 GEMM's A image
/// (tc_bf16x3_a_bytes layout: 128-row tiles x 32-column chunks x hi | lo x
/// 128 rows x 64 B, SWIZZLE_64B rows; a = hi + lo, hi = bf16(a), lo =
/// bf16(a - hi) — the split kernel's arithmetic), 8-value groups.
__device__ __forceinline__ void bf16_rows(const float* src, int lds, int rows, int K, std::size_t b0,
                                          unsigned char* img) {
    const int nch = (K + 31) / 32, groups = nch * 4;
    int r = threadIdx.x / groups, kg = threadIdx.x - r * groups;
    for (; r < rows; step_rk(r, kg, kThreads, groups)) {
        const int k0 = 8 * kg;
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = k0 + u < K ? src[r * lds + k0 + u] : 0.f;
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float h0 = __bfloat162float(__float2bfloat16_rn(v[2 * q]));
            const float h1 = __bfloat162float(__float2bfloat16_rn(v[2 * q + 1]));
            hi[q] = bf16_pair(h0, h1);
            lo[q] = bf16_pair(v[2 * q] - h0, v[2 * q + 1] - h1);
        }
        const std::size_t grow = b0 + r;
        unsigned char* blk = img + ((grow >> 7) * nch + (k0 >> 5)) * 16384 + sw64_int8(static_cast<int>(grow & 127),
                                                                                         (k0 & 31) >> 3);
        *reinterpret_cast<uint4*>(blk) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(blk + 8192) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
}

/// FOLD (antisymmetric plans): the input rows hold 2n samples; the kernel
/// writes u_j = x_j - x_{2n-1-j} to `hat` and transforms y_j = x_j + x_{2n-1-j}
/// (length n), whose DCT gives the even coefficients of the full row.  With
/// fs.sl set (fp64), u is not written: it stays in shared memory and leaves as
/// the int8 slices of the W product (ozaki.cu's digits and tile image), so the
/// product needs no separate slicing pass over u.
template <class T, bool FOLD = false>
__global__ void __launch_bounds__(kThreads)
dct2_fft_kernel(const T* __restrict__ in, std::size_t ld_in, T* __restrict__ hat, std::size_t ld_hat,
                T* __restrict__ out, std::size_t ld_out, Emit<T> emit, int n, int logn,
                int rows_per_cta, std::size_t batch, Twiddles<T> tw, int* flag, FoldSlices fs) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = n >> 1, logN = logn - 1, ld = padded_len(N);
    cplx_t<T>* nat = reinterpret_cast<cplx_t<T>*>(smem_raw);
    cplx_t<T>* work = nat + rows_per_cta * ld;
    T* sh = reinterpret_cast<T*>(nat); // real output rows (stride n) once `nat` is consumed
    T* ush = reinterpret_cast<T*>(work + rows_per_cta * ld); // u rows (fs.sl), then row maxima
    const bool slice = FOLD && sizeof(T) == 8 && fs.sl != nullptr;
    const bool tobf = FOLD && sizeof(T) == 4 && fs.bf != nullptr; // u -> the bf16x3 A image (fp32)
    const bool to_smem = slice || tobf;                            // u rows stay in shared memory
    const std::size_t b0 = static_cast<std::size_t>(blockIdx.x) * rows_per_cta;
    const int rows = static_cast<int>(min(static_cast<std::size_t>(rows_per_cta), batch - b0));

    // Load with Makhoul's permutation v = (x0, x2, ..., x3, x1), packed as
    // w_m = v_{2m} + i v_{2m+1}, in natural order (the FFT's first pass does
    // the bit reversal).  Eight independent loads in flight per thread
    // before any use (a load-use chain per element left the kernel waiting on
    // HBM latency).
    bool bad = false;
    constexpr int U = 8;
    // 16-byte rows: four consecutive samples (and their four mirrors) per
    // thread step, vector loads and stores; Makhoul pairs (j, j+2) and
    // (j+3, j+1) each become one complex store
    // (fp64: two steps in flight per thread — four measured slower, 0.105 -> 0.123 ms at C3)
    const bool vec4 = n % 4 == 0 && reinterpret_cast<std::uintptr_t>(in) % 16 == 0 && (ld_in * sizeof(T)) % 16 == 0 &&
                      (to_smem || !FOLD || (reinterpret_cast<std::uintptr_t>(hat) % 16 == 0 && (ld_hat * sizeof(T)) % 16 == 0));
    if (vec4) {
        constexpr int U4 = sizeof(T) == 8 ? 2 : 4;
        const int n4 = n >> 2, logn4 = logn - 2;
        for (int t0 = threadIdx.x; t0 < rows * n4; t0 += U4 * kThreads) {
            T xv[U4][4], xm[U4][4];
#pragma unroll
            for (int u = 0; u < U4; ++u) {
                const int t = t0 + u * kThreads;
                if (t < rows * n4) {
                    const T* row = in + (b0 + (t >> logn4)) * ld_in;
                    const int j0 = 4 * (t & (n4 - 1));
                    load4(row + j0, xv[u]);
                    if constexpr (FOLD) load4(row + 2 * n - 4 - j0, xm[u]); // reversed below
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) xv[u][q] = xm[u][q] = T(0);
                }
            }
#pragma unroll
            for (int u = 0; u < U4; ++u) {
                const int t = t0 + u * kThreads;
                if (t >= rows * n4) break;
                const int r = t >> logn4, j0 = 4 * (t & (n4 - 1));
                T v[4], uu[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    bad |= !finite_val(xv[u][q]);
                    v[q] = xv[u][q];
                    if constexpr (FOLD) {
                        const T m = xm[u][3 - q]; // x_{2n-1-(j0+q)}
                        bad |= !finite_val(m);
                        uu[q] = v[q] - m;
                        v[q] = v[q] + m;
                    }
                }
                if constexpr (FOLD) {
                    if (to_smem)
                        store4(ush + r * n + j0, uu);
                    else
                        store4(hat + (b0 + r) * ld_hat + j0, uu);
                }
                nat[r * ld + pad8(j0 >> 2)] = cplx_t<T>{v[0], v[2]};
                nat[r * ld + pad8(N - 1 - (j0 >> 2))] = cplx_t<T>{v[3], v[1]};
            }
        }
    } else
    for (int t0 = threadIdx.x; t0 < rows * n; t0 += U * kThreads) {
        T xv[U], xm[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = t0 + u * kThreads;
            const std::size_t row = (b0 + (t >> logn)) * ld_in;
            xv[u] = t < rows * n ? in[row + (t & (n - 1))] : T(0);
            if constexpr (FOLD) xm[u] = t < rows * n ? in[row + 2 * n - 1 - (t & (n - 1))] : T(0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = t0 + u * kThreads;
            if (t >= rows * n) break;
            const int r = t >> logn, j = t & (n - 1);
            bad |= !finite_val(xv[u]);
            T v = xv[u];
            if constexpr (FOLD) {
                bad |= !finite_val(xm[u]);
                if (to_smem)
                    ush[r * n + j] = xv[u] - xm[u];
                else
                    hat[(b0 + r) * ld_hat + j] = xv[u] - xm[u];
                v = xv[u] + xm[u];
            }
            const int p = (j & 1) ? (n - 1 - (j >> 1)) : (j >> 1);
            reinterpret_cast<T*>(&nat[r * ld + pad8(p >> 1)])[p & 1] = v;
        }
    }
    if (bad) atomicOr(flag, 1);
    __syncthreads();

    if constexpr (FOLD && sizeof(T) == 4) {
        if (tobf) bf16_rows(reinterpret_cast<const float*>(ush), n, rows, n, b0, fs.bf);
    }
    if constexpr (FOLD) {
        if (slice) { // u -> int8 digits (ozaki_slice_kernel's arithmetic), per row
            double* rmax = reinterpret_cast<double*>(ush + rows * n);
            const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
            for (int r = warp; r < rows; r += kThreads / 32) {
                double mx = 0.0;
                bool nf = false;
                for (int j = lane; j < n; j += 32) {
                    const double v = static_cast<double>(ush[r * n + j]);
                    nf |= !isfinite(v);
                    mx = fmax(mx, fabs(v));
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                if (__any_sync(0xffffffffu, nf)) mx = 0.0; // flagged above
                if (lane == 0) {
                    int e = 0;
                    if (mx > 0.0) frexp(mx, &e);
                    fs.expo[b0 + r] = e;
                    rmax[r] = ldexp(127.0, -e);
                }
            }
            __syncthreads();
            slice_rows(reinterpret_cast<const double*>(ush), n, rows, n, b0, fs, rmax);
        }
    }

    fft_rows<T, false>(nat, work, rows, N, logN, tw.fft);

    // Real split V_k = E_k - i e^{-2 pi i k/n} O_k, then Y_k = Re(e^{-i pi k/2n} V_k),
    // Y_{n-k} = -Im(...); orthonormal scale sqrt(2/n), DC gets 1/sqrt(2) more.
    const T scale = static_cast<T>(sqrt(2.0 / n));
    const T dc_scale = static_cast<T>(1.0 / sqrt(static_cast<double>(n)));
    const T half = static_cast<T>(0.5);
    for (int t = threadIdx.x; t < rows * N; t += blockDim.x) {
        const int r = t >> logN, k = t & (N - 1);
        const cplx_t<T>* row = work + r * ld;
        T* o = sh + r * n;
        if (k == 0) {
            const cplx_t<T> w0 = row[0];
            o[0] = (w0.x + w0.y) * dc_scale;
            o[N] = (w0.x - w0.y) * __ldg(tw.rot + 2 * N) * scale;
            continue;
        }
        const cplx_t<T> wk = row[pad8(k)];
        const cplx_t<T> wc = row[pad8(N - k)];
        const T er = half * (wk.x + wc.x), ei = half * (wk.y - wc.y);
        const T orr = half * (wk.x - wc.x), oi = half * (wk.y + wc.y);
        const cplx_t<T> sp = __ldg(reinterpret_cast<const cplx_t<T>*>(tw.split) + k);
        const T sr = sp.x, si = sp.y;
        const T qr = sr * orr - si * oi, qi = sr * oi + si * orr;
        const T vr = er + qi, vi = ei - qr;
        const cplx_t<T> rt = __ldg(reinterpret_cast<const cplx_t<T>*>(tw.rot) + k);
        const T cr = rt.x, ci = rt.y;
        o[k] = (vr * cr - vi * ci) * scale;
        o[n - k] = -(vr * ci + vi * cr) * scale;
    }
    __syncthreads();

    if (!FOLD && hat != nullptr)
        for (int t = threadIdx.x; t < rows * n; t += blockDim.x) {
            const int r = t >> logn, k = t & (n - 1);
            hat[(b0 + r) * ld_hat + k] = sh[t];
        }
    // one table lookup per entry, reused for every row of the tile
    for (int e = threadIdx.x; e < emit.count; e += blockDim.x) {
        const int to = __ldg(emit.to + e), from = __ldg(emit.from + e);
        const T sg = __ldg(emit.sign + e);
        for (int r = 0; r < rows; ++r) {
            const T v = sg * sh[r * n + from];
            if (to >= 0)
                out[(b0 + r) * ld_out + to] = v;
            else
                emit.alt[(b0 + r) * emit.ld_alt + (-to - 1)] = v;
        }
    }
}

/// Digits of K gathered values per row (ozaki.cu's slicing arithmetic and
/// tile image), rows b0.. of a CTA: g holds the rows' values (stride K),
/// rmax scratch per row.
__device__ void slice_rows_to_tiles(const double* g, int rows, int K, std::size_t b0, const FoldSlices& fs,
                                    double* rmax) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int r = warp; r < rows; r += kThreads / 32) {
        double mx = 0.0;
        bool nf = false;
        for (int j = lane; j < K; j += 32) {
            nf |= !isfinite(g[r * K + j]);
            mx = fmax(mx, fabs(g[r * K + j]));
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (__any_sync(0xffffffffu, nf)) mx = 0.0;
        if (lane == 0) {
            int e = 0;
            if (mx > 0.0) frexp(mx, &e);
            fs.expo[b0 + r] = e;
            rmax[r] = ldexp(127.0, -e);
        }
    }
    __syncthreads();
    slice_rows(g, K, rows, K, b0, fs, rmax);
}

/// fs.sl set (fp64): the K = fs.K values p[row, fs.map[k]] of each row also
/// leave as the int8 slices of the folded inverse's W product (no separate
/// gather-and-slice pass over p).
template <class T>
__global__ void __launch_bounds__(kThreads)
idct_fft_kernel(const T* __restrict__ d, std::size_t ld_d, const T* __restrict__ p, std::size_t ld_p,
                Emit<T> emit, T* __restrict__ out, std::size_t ld_out, int n, int logn,
                int rows_per_cta, std::size_t batch, Twiddles<T> tw, int* flag, FoldSlices fs) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = n >> 1, logN = logn - 1, ld = padded_len(N);
    cplx_t<T>* nat = reinterpret_cast<cplx_t<T>*>(smem_raw);
    cplx_t<T>* work = nat + rows_per_cta * ld;
    T* sh = reinterpret_cast<T*>(work); // the real coefficients, consumed before the FFT writes `work`
    const std::size_t b0 = static_cast<std::size_t>(blockIdx.x) * rows_per_cta;
    const int rows = static_cast<int>(min(static_cast<std::size_t>(rows_per_cta), batch - b0));
    // The folded inverse (zero d rows, p's W slots gathered for the product):
    // both gathers from p — the W slots into g, the even slots into the
    // IDCT input — with all their loads in flight together (one global
    // round trip per CTA instead of two), then the W slots leave as the
    // product's A image (int8 digits in fp64, bf16 halves in fp32).
    const bool comb = !d && ((sizeof(T) == 8 && fs.sl != nullptr) || (sizeof(T) == 4 && fs.bf != nullptr));
    if (comb) {
        for (int t = threadIdx.x; t < (rows * n * static_cast<int>(sizeof(T))) / 16; t += kThreads)
            reinterpret_cast<uint4*>(sh)[t] = make_uint4(0u, 0u, 0u, 0u);
        __syncthreads();
        T* g = reinterpret_cast<T*>(work + rows_per_cta * ld);
        constexpr int U = 8;
        const int tot_o = rows * fs.K, tot_e = rows * emit.count;
        int r0 = threadIdx.x / fs.K, k0 = threadIdx.x - r0 * fs.K;
        int re = emit.count > 0 ? threadIdx.x / emit.count : rows, ee = emit.count > 0 ? threadIdx.x - re * emit.count : 0;
        bool nf = false;
        for (int t0 = 0; t0 < max(tot_o, tot_e); t0 += U * kThreads) {
            T vo[U], ve[U];
            int ri[U], ei[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                vo[u] = r0 < rows ? p[(b0 + r0) * ld_p + __ldg(fs.map + k0)] : T(0);
                step_rk(r0, k0, kThreads, fs.K);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                ri[u] = re;
                ei[u] = ee;
                ve[u] = re < rows ? p[(b0 + re) * ld_p + __ldg(emit.from + ee)] : T(0);
                if (emit.count > 0) step_rk(re, ee, kThreads, emit.count);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = t0 + u * kThreads + static_cast<int>(threadIdx.x);
                if (t < tot_o) {
                    nf |= !finite_val(vo[u]);
                    g[t] = vo[u];
                }
                if (ri[u] < rows) {
                    nf |= !finite_val(ve[u]);
                    sh[ri[u] * n + __ldg(emit.to + ei[u])] = __ldg(emit.sign + ei[u]) * ve[u];
                }
            }
        }
        if (nf) atomicOr(flag, 1);
        __syncthreads();
        if constexpr (sizeof(T) == 8)
            slice_rows_to_tiles(reinterpret_cast<const double*>(g), rows, fs.K, b0, fs,
                                reinterpret_cast<double*>(g) + rows_per_cta * fs.K);
        else
            bf16_rows(reinterpret_cast<const float*>(g), fs.K, rows, fs.K, b0, fs.bf);
    }
    if constexpr (sizeof(T) == 8) {
        if (fs.sl != nullptr && !comb) { // gathered values into the extra shared rows, then their digits
            double* g = reinterpret_cast<double*>(work + rows_per_cta * ld);
            double* rmax = g + rows_per_cta * fs.K;
            constexpr int U = 8;
            bool nf = false;
            int r0 = threadIdx.x / fs.K, k0 = threadIdx.x - r0 * fs.K;
            for (int t0 = threadIdx.x; t0 < rows * fs.K; t0 += U * kThreads) {
                double v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (r0 < rows) {
                        v[u] = static_cast<double>(p[(b0 + r0) * ld_p + __ldg(fs.map + k0)]);
                    } else {
                        v[u] = 0.0;
                    }
                    step_rk(r0, k0, kThreads, fs.K);
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (t0 + u * kThreads < rows * fs.K) {
                        nf |= !isfinite(v[u]);
                        g[t0 + u * kThreads] = v[u];
                    }
            }
            if (nf) atomicOr(flag, 1);
            __syncthreads();
            slice_rows_to_tiles(g, rows, fs.K, b0, fs, rmax);
        }
    }

    if constexpr (sizeof(T) == 4) {
        if (fs.bf != nullptr && !comb) { // gathered W slots -> the bf16x3 A image (no gathered split pass)
            float* g = reinterpret_cast<float*>(work + rows_per_cta * ld);
            constexpr int U = 8;
            bool nf = false;
            int r0 = threadIdx.x / fs.K, k0 = threadIdx.x - r0 * fs.K;
            for (int t0 = threadIdx.x; t0 < rows * fs.K; t0 += U * kThreads) {
                float v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    v[u] = r0 < rows ? p[(b0 + r0) * ld_p + __ldg(fs.map + k0)] : 0.f;
                    step_rk(r0, k0, kThreads, fs.K);
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (t0 + u * kThreads < rows * fs.K) {
                        nf |= !isfinite(v[u]);
                        g[t0 + u * kThreads] = v[u];
                    }
            }
            if (nf) atomicOr(flag, 1);
            __syncthreads();
            bf16_rows(g, fs.K, rows, fs.K, b0, fs.bf);
        }
    }

    // X_k = sqrt(2/n) c_k d_k, with X_0 doubled (the REDFT01 convention).
    const T scale = static_cast<T>(sqrt(2.0 / n));
    const T dc_scale = static_cast<T>(2.0 / sqrt(static_cast<double>(n)));
    constexpr int U = 8; // independent loads in flight per thread
    if (comb) {
        // sh already holds the even slots (above)
    } else if (!d) { // zero d rows (the folded inverse): plain 16-byte zero stores
        for (int t = threadIdx.x; t < (rows * n * static_cast<int>(sizeof(T))) / 16; t += kThreads)
            reinterpret_cast<uint4*>(sh)[t] = make_uint4(0u, 0u, 0u, 0u);
    } else
    for (int t0 = threadIdx.x; t0 < rows * n; t0 += U * kThreads) {
        T v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = t0 + u * kThreads;
            v[u] = t < rows * n ? d[(b0 + (t >> logn)) * ld_d + (t & (n - 1))] : T(0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (t0 + u * kThreads < rows * n) sh[t0 + u * kThreads] = v[u];
    }
    __syncthreads();
    bool bad = false;
    if (emit.count > 0 && !comb) {
        int re = threadIdx.x / emit.count, ee = threadIdx.x - re * emit.count;
        for (int t0 = threadIdx.x; t0 < rows * emit.count; t0 += U * kThreads) {
            T v[U];
            int ri[U], ei[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                ri[u] = re;
                ei[u] = ee;
                v[u] = re < rows ? p[(b0 + re) * ld_p + __ldg(emit.from + ee)] : T(0);
                step_rk(re, ee, kThreads, emit.count);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (ri[u] >= rows) break;
                bad |= !finite_val(v[u]);
                sh[ri[u] * n + __ldg(emit.to + ei[u])] = __ldg(emit.sign + ei[u]) * v[u];
            }
        }
    }
    if (bad) atomicOr(flag, 1);
    __syncthreads();
    for (int t = threadIdx.x; t < rows * n; t += blockDim.x) sh[t] *= ((t & (n - 1)) == 0) ? dc_scale : scale;
    __syncthreads();

    // V_k = e^{i pi k/2n} (X_k - i X_{n-k}); Z_k = (V_k + V_{k+N} + i e^{2 pi i k/n}(V_k - V_{k+N}))/2,
    // stored in natural order (the FFT's first pass gathers bit-reversed)
    const T half = static_cast<T>(0.5);
    const T r2 = static_cast<T>(0.70710678118654752440);
    for (int t = threadIdx.x; t < rows * N; t += blockDim.x) {
        const int r = t >> logN, k = t & (N - 1);
        const T* x = sh + r * n;
        const cplx_t<T> rt = __ldg(reinterpret_cast<const cplx_t<T>*>(tw.rot) + k);
        const T cr = rt.x, ci = -rt.y; // e^{+i pi k/2n}
        const T ar = x[k], ai = (k == 0) ? T(0) : -x[n - k];
        const T v1r = ar * cr - ai * ci, v1i = ar * ci + ai * cr;
        // e^{i pi (k+N)/2n} = e^{i pi/4} e^{i pi k/2n}
        const T c2r = r2 * (cr - ci), c2i = r2 * (cr + ci);
        const T br = x[k + N], bi = -x[N - k];
        const T v2r = br * c2r - bi * c2i, v2i = br * c2i + bi * c2r;
        const cplx_t<T> sp = __ldg(reinterpret_cast<const cplx_t<T>*>(tw.split) + k);
        const T sr = sp.x, si = -sp.y; // e^{+2 pi i k/n}
        const T dr = v1r - v2r, di = v1i - v2i;
        const T qr = sr * dr - si * di, qi = sr * di + si * dr;
        nat[r * ld + pad8(k)] = {half * (v1r + v2r - qi), half * (v1i + v2i + qr)};
    }
    __syncthreads();

    fft_rows<T, true>(nat, work, rows, N, logN, tw.fft);

    for (int t = threadIdx.x; t < rows * n; t += blockDim.x) {
        const int r = t >> logn, j = t & (n - 1);
        const int pidx = (j & 1) ? (n - 1 - (j >> 1)) : (j >> 1);
        const cplx_t<T> w = work[r * ld + pad8(pidx >> 1)];
        out[(b0 + r) * ld_out + j] = (pidx & 1) ? w.y : w.x;
    }
}

// --- any n: direct O(n^2) over the cos(pi m / 2n) table ------------------------

template <class T>
__global__ void __launch_bounds__(kThreads)
dct2_direct_kernel(const T* __restrict__ in, std::size_t ld_in, T* __restrict__ hat, std::size_t ld_hat,
                   T* __restrict__ out, std::size_t ld_out, Emit<T> emit, int n, std::size_t batch,
                   Twiddles<T> tw, int* flag) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* x = reinterpret_cast<T*>(smem_raw);
    T* o = x + n;
    const std::size_t b = blockIdx.x;
    bool bad = false;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        x[j] = in[b * ld_in + j];
        bad |= !finite_val(x[j]);
    }
    if (bad) atomicOr(flag, 1);
    __syncthreads();
    const int m4 = 4 * n;
    const T scale = static_cast<T>(sqrt(2.0 / n));
    const T dc_scale = static_cast<T>(1.0 / sqrt(static_cast<double>(n)));
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        T acc = 0;
        int idx = k % m4, inc = (2 * k) % m4;
        for (int j = 0; j < n; ++j) {
            acc += x[j] * __ldg(tw.cos4n + idx);
            idx += inc;
            if (idx >= m4) idx -= m4;
        }
        o[k] = acc * (k == 0 ? dc_scale : scale);
    }
    __syncthreads();
    if (hat != nullptr)
        for (int k = threadIdx.x; k < n; k += blockDim.x) hat[b * ld_hat + k] = o[k];
    for (int e = threadIdx.x; e < emit.count; e += blockDim.x) {
        const int to = emit.to[e];
        const T v = emit.sign[e] * o[emit.from[e]];
        if (to >= 0)
            out[b * ld_out + to] = v;
        else
            emit.alt[b * emit.ld_alt + (-to - 1)] = v;
    }
}

template <class T>
__global__ void __launch_bounds__(kThreads)
idct_direct_kernel(const T* __restrict__ d, std::size_t ld_d, const T* __restrict__ p, std::size_t ld_p,
                   Emit<T> emit, T* __restrict__ out, std::size_t ld_out, int n, std::size_t batch,
                   Twiddles<T> tw, int* flag) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* x = reinterpret_cast<T*>(smem_raw);
    const std::size_t b = blockIdx.x;
    for (int k = threadIdx.x; k < n; k += blockDim.x) x[k] = d[b * ld_d + k];
    __syncthreads();
    bool bad = false;
    for (int e = threadIdx.x; e < emit.count; e += blockDim.x) {
        const T v = p[b * ld_p + emit.from[e]];
        bad |= !finite_val(v);
        x[emit.to[e]] = emit.sign[e] * v;
    }
    if (bad) atomicOr(flag, 1);
    __syncthreads();
    const int m4 = 4 * n;
    const T scale = static_cast<T>(sqrt(2.0 / n));
    const T dc_scale = static_cast<T>(1.0 / sqrt(static_cast<double>(n)));
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        T acc = x[0] * dc_scale;
        const int inc = (2 * j + 1) % m4;
        int idx = inc;
        for (int k = 1; k < n; ++k) {
            acc += x[k] * scale * __ldg(tw.cos4n + idx);
            idx += inc;
            if (idx >= m4) idx -= m4;
        }
        out[b * ld_out + j] = acc;
    }
}

template <class T>
int rows_per_cta_for(std::size_t n) {
    return static_cast<int>(std::max<std::size_t>(1, kTileElems / n));
}

} // namespace

template <class T>
cudaError_t dct2_rows(const T* in, std::size_t ld_in, T* hat, std::size_t ld_hat, T* out,
                      std::size_t ld_out, Emit<T> emit, std::size_t n, std::size_t batch,
                      Twiddles<T> tw, int* flag, cudaStream_t stream) {
    if (batch == 0) return cudaSuccess;
    if (is_pow2(n) && n >= 2) {
        const int rows = rows_per_cta_for<T>(n);
        const std::size_t smem = fft_smem_bytes<T>(n, rows);
        auto kern = dct2_fft_kernel<T>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        const unsigned grid = static_cast<unsigned>((batch + rows - 1) / rows);
        kern<<<grid, kThreads, smem, stream>>>(in, ld_in, hat, ld_hat, out, ld_out, emit,
                                              static_cast<int>(n), ilog2(n), rows, batch, tw, flag, FoldSlices{});
        return cudaGetLastError();
    }
    const std::size_t smem = 2 * n * sizeof(T);
    auto kern = dct2_direct_kernel<T>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(batch), kThreads, smem, stream>>>(in, ld_in, hat, ld_hat, out, ld_out, emit,
                                                                 static_cast<int>(n), batch, tw, flag);
    return cudaGetLastError();
}

template <class T>
cudaError_t dct2_fold_rows(const T* in, std::size_t ld_in, T* u, std::size_t ld_u, T* out, std::size_t ld_out,
                           Emit<T> emit, std::size_t n, std::size_t batch, Twiddles<T> tw, int* flag,
                           cudaStream_t stream, FoldSlices fs) {
    if (batch == 0) return cudaSuccess;
    if (!is_pow2(n) || n < 2) return cudaErrorInvalidValue;
    if ((fs.sl && sizeof(T) != 8) || (fs.bf && sizeof(T) != 4)) return cudaErrorInvalidValue;
    const int rows = rows_per_cta_for<T>(n);
    const std::size_t smem = fft_smem_bytes<T>(n, rows) +
                             ((fs.sl || fs.bf) ? static_cast<std::size_t>(rows) * (n * sizeof(T) + sizeof(double)) : 0);
    auto kern = dct2_fft_kernel<T, true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const unsigned grid = static_cast<unsigned>((batch + rows - 1) / rows);
    kern<<<grid, kThreads, smem, stream>>>(in, ld_in, u, ld_u, out, ld_out, emit, static_cast<int>(n), ilog2(n), rows,
                                          batch, tw, flag, fs);
    return cudaGetLastError();
}

template <class T>
cudaError_t idct_rows(const T* d, std::size_t ld_d, const T* p, std::size_t ld_p, Emit<T> emit,
                      T* out, std::size_t ld_out, std::size_t n, std::size_t batch,
                      Twiddles<T> tw, int* flag, cudaStream_t stream, FoldSlices fs) {
    if (batch == 0) return cudaSuccess;
    if (is_pow2(n) && n >= 2) {
        const int rows = rows_per_cta_for<T>(n);
        if ((fs.sl && sizeof(T) != 8) || (fs.bf && sizeof(T) != 4)) return cudaErrorInvalidValue;
        const std::size_t smem =
            fft_smem_bytes<T>(n, rows) +
            (fs.sl ? static_cast<std::size_t>(rows) * (static_cast<std::size_t>(fs.K) + 1) * sizeof(double) : 0) +
            (fs.bf ? static_cast<std::size_t>(rows) * static_cast<std::size_t>(fs.K) * sizeof(float) : 0);
        auto kern = idct_fft_kernel<T>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        const unsigned grid = static_cast<unsigned>((batch + rows - 1) / rows);
        kern<<<grid, kThreads, smem, stream>>>(d, ld_d, p, ld_p, emit, out, ld_out, static_cast<int>(n),
                                              ilog2(n), rows, batch, tw, flag, fs);
        return cudaGetLastError();
    }
    if (!d) return cudaErrorInvalidValue; // zero d rows (d = nullptr): the FFT kernel only
    const std::size_t smem = n * sizeof(T);
    auto kern = idct_direct_kernel<T>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(batch), kThreads, smem, stream>>>(d, ld_d, p, ld_p, emit, out, ld_out,
                                                                 static_cast<int>(n), batch, tw, flag);
    return cudaGetLastError();
}

bool dct_supported(std::size_t n, bool f64) {
    constexpr std::size_t kSmemMax = 227 * 1024;
    if (n < 1) return false;
    if (is_pow2(n) && n >= 2) {
        const std::size_t smem = f64 ? fft_smem_bytes<double>(n, rows_per_cta_for<double>(n))
                                     : fft_smem_bytes<float>(n, rows_per_cta_for<float>(n));
        return smem <= kSmemMax;
    }
    return 2 * n * (f64 ? sizeof(double) : sizeof(float)) <= kSmemMax;
}

template cudaError_t dct2_rows<double>(const double*, std::size_t, double*, std::size_t, double*, std::size_t,
                                       Emit<double>, std::size_t, std::size_t, Twiddles<double>, int*, cudaStream_t);
template cudaError_t dct2_rows<float>(const float*, std::size_t, float*, std::size_t, float*, std::size_t,
                                      Emit<float>, std::size_t, std::size_t, Twiddles<float>, int*, cudaStream_t);
template cudaError_t dct2_fold_rows<double>(const double*, std::size_t, double*, std::size_t, double*, std::size_t,
                                            Emit<double>, std::size_t, std::size_t, Twiddles<double>, int*,
                                            cudaStream_t, FoldSlices);
template cudaError_t dct2_fold_rows<float>(const float*, std::size_t, float*, std::size_t, float*, std::size_t,
                                           Emit<float>, std::size_t, std::size_t, Twiddles<float>, int*, cudaStream_t,
                                           FoldSlices);
template cudaError_t idct_rows<double>(const double*, std::size_t, const double*, std::size_t, Emit<double>,
                                       double*, std::size_t, std::size_t, std::size_t, Twiddles<double>, int*,
                                       cudaStream_t, FoldSlices);
template cudaError_t idct_rows<float>(const float*, std::size_t, const float*, std::size_t, Emit<float>, float*,
                                      std::size_t, std::size_t, std::size_t, Twiddles<float>, int*, cudaStream_t,
                                      FoldSlices);

} // namespace dctp::dev
