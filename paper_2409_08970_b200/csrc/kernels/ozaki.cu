// fp64 products on the int8 tensor cores (tcgen05 kind::i8), sm_100a:
//
//   out[b, c] = sum_k in[b, k] * bt[c, k]          (bt = X^T, or X, or W^T)
//
// the dense routes' X^T s / X p (C5: fast_transform.hpp:199-214, the route
// the reference's near-pole guard sends config 5 to) and the rank-k chain
// apply, which on the DMMA pipe are capped at the 37 TF/s fp64 tensor rate.
//
// Ozaki-style slicing.  Each row r of either operand is scaled by a power of
// two, 2^-e_r with max_k |x_rk| < 2^e_r, and written as S int8 digits:
//   x_rk 2^-e_r = (d_0 + d_1/254 + ... + d_{S-1}/254^{S-1}) / 127 + residual,
// d_0 = rint(127 x 2^-e) and every later digit the rounded residual times 254,
// all in [-127, 127] (|residual| <= 1/2 before each scaling).  The product is
// then a sum of integer products
//   sum_k x_bk y_ck = 2^(e_b + f_c) / 127^2 * sum_L 254^-L D_L,
//   D_L = sum_{i + j = L} sum_k d^x_i[b,k] d^y_j[c,k]
// where every D_L is exact in int32 (|D_L| <= (L+1) K 127^2 < 2^31 for K up to
// 2^16 / (L+1)).  Keeping the levels L <= LMAX (LMAX = S - 1: S(S+1)/2 integer
// GEMMs) bounds the error by the dropped tail; measured on C5 (n = 8192, the
// reference's own basis): 2.5e-11 for S = 5 (15 products) and 9e-14 for S = 6
// (21 products), norm-wise per signal, against the 1e-10 fp64 tolerance.
//
// GEMM kernel: one CTA per 128 x NT output tile (non-persistent: K is long,
// the epilogue is ~2% of a tile), 128 threads.  Every level has its own int32
// accumulator in TMEM ((LMAX + 1) * NT <= 512 columns).  Operands arrive
// pre-sliced in the exact shared-memory image (per tile and 64-byte K chunk:
// S slices of 128 (A) or NT (B) rows x 64 bytes, K-major SWIZZLE_64B) by two
// TMA bulk copies per stage into a multi-stage mbarrier ring; lane 0 of warp 0
// produces, lane 0 of warp 1 issues the S(S+1)/2 MMAs of each 32-byte K step
// and commits the stage back to the producer; at the end all four warps read
// their 32 TMEM lanes level by level (Horner in fp64, exact int32 -> fp64
// conversions), scale by 2^(e_b + f_c) / 127^2 and store the fp64 rows.
#include <cstdint>
#include <cstdlib>

#include "kernels/common.cuh"
#include "kernels/launch.hpp"

namespace dctp::dev {
namespace {

constexpr int CB = 64;          // K chunk: 64 int8 = one SWIZZLE_64B atom row
constexpr int TM = 128;         // A tile rows (TMEM lanes)
constexpr int kThreads = 128;
constexpr int kMaxSmem = 227 * 1024;

__device__ __forceinline__ uint32_t sw64(int r, int c16) {
    return static_cast<uint32_t>(r * 64 + ((c16 ^ ((r >> 1) & 3)) << 4));
}

/// K-major SWIZZLE_64B shared-memory descriptor (8-row groups of 512 bytes).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(512 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(4) << 61;
    return d;
}

/// D s32, A and B signed int8, both K-major, M = 128, N = NT.
template <int NT>
__host__ __device__ constexpr uint32_t idesc_i8() {
    return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(NT >> 3) << 17) |
           (static_cast<uint32_t>(TM >> 4) << 24);
}

template <int NT>
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc_i8<NT>()), "r"(accumulate));
}

/// One lane of a converged warp (elect.sync): the warp-uniform issue pattern
/// that keeps the MMA loop in uniform registers.
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}\n" : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     ptx::smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

// ---------------------------------------------------------------- slicing

/// Slicing of one row per WPR warps (WPR = 8: a CTA per row, long rows;
/// WPR = 1: a warp per row, 8 rows per CTA, rows up to 2048): pass 1 the row
/// maximum (and the finiteness check of check_signal), pass 2 the S digits.
/// Thread t handles 4 consecutive k per step (one 32-bit word of a 16-byte
/// swizzle unit), so both passes read the row with coalesced 32-byte loads
/// (vec: 16-byte aligned rows, no column map) and each slice's 64-byte chunk
/// rows are written as whole sectors; pass 2 finds the row in L1/L2.
template <class T, int WPR>
__global__ void __launch_bounds__(256)
ozaki_slice_kernel(const T* __restrict__ in, std::size_t ld, std::size_t rows, std::size_t rows_pad, int K, int nch,
                   const int* __restrict__ a_map, int tile_rows, int S, int8_t* __restrict__ sl,
                   int* __restrict__ expo, int* flag, int vec) {
    constexpr int kRowThreads = 32 * WPR;
    __shared__ double red[8];
    __shared__ int red_bad[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = WPR == 8 ? static_cast<int>(threadIdx.x) : lane; // thread index within the row
    const std::size_t r = WPR == 8 ? blockIdx.x : static_cast<std::size_t>(blockIdx.x) * 8 + warp;
    if (r >= rows_pad) return; // whole warps (WPR = 1) or whole CTAs (WPR = 8)
    const bool real = r < rows;
    const T* row = in + (real ? r * ld : 0);
    auto load4 = [&](int k, double (&v)[4]) {
        if (real && vec && k + 3 < K) {
            if constexpr (sizeof(T) == 8) {
                const double2 a = __ldg(reinterpret_cast<const double2*>(row + k));
                const double2 b = __ldg(reinterpret_cast<const double2*>(row + k + 2));
                v[0] = a.x, v[1] = a.y, v[2] = b.x, v[3] = b.y;
            } else {
                const float4 a = __ldg(reinterpret_cast<const float4*>(row + k));
                v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
            }
            return;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            v[u] = (real && k + u < K) ? static_cast<double>(row[a_map ? __ldg(a_map + k + u) : k + u]) : 0.0;
    };
    double mx = 0.0;
    bool bad = false;
#pragma unroll 2
    for (int k = 4 * t; k < K; k += 4 * kRowThreads) {
        double v[4];
        load4(k, v);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            bad |= !isfinite(v[u]);
            mx = fmax(mx, fabs(v[u]));
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int anybad = __any_sync(0xffffffffu, bad);
    if constexpr (WPR == 8) {
        if (lane == 0) {
            red[warp] = mx;
            red_bad[warp] = anybad;
        }
        __syncthreads();
        mx = red[0];
        anybad = red_bad[0];
#pragma unroll
        for (int w = 1; w < 8; ++w) {
            mx = fmax(mx, red[w]);
            anybad |= red_bad[w];
        }
    }
    if (anybad) {
        if (t == 0 && flag) atomicOr(flag, 1);
        mx = 0.0;
    }
    int e = 0;
    if (mx > 0.0) frexp(mx, &e); // mx = m 2^e, m in [0.5, 1): |x| < 2^e
    if (t == 0) expo[r] = e;
    const double scale = ldexp(127.0, -e);
    const std::size_t tile = r / tile_rows;
    const int lr = static_cast<int>(r % tile_rows);
    const std::size_t slice_bytes = static_cast<std::size_t>(tile_rows) * CB;
#pragma unroll 2
    for (int k = 4 * t; k < nch * CB; k += 4 * kRowThreads) {
        double v[4];
        load4(k, v);
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = isfinite(v[u]) ? v[u] * scale : 0.0;
        const int ch = k / CB, c16 = (k % CB) / 16;
        int8_t* dst = sl + ((tile * nch + ch) * S) * slice_bytes + sw64(lr, c16) + (k % 16);
        for (int s = 0; s < S; ++s) {
            uint32_t w = 0u;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                w |= ozaki_digit(v[u]) << (8 * u);
            }
            *reinterpret_cast<uint32_t*>(dst + s * slice_bytes) = w;
        }
    }
}

/// Long fp64 rows (2048 < K <= 8192, 16-byte aligned, no column map: C5's
/// signals): one CTA per row keeps the row in registers (thread t: 8-value
/// groups k = 8 t + 2048 i), so it is read once — all loads in flight before
/// the maximum — and each group leaves as one 8-byte store per slice plane.
template <int S, int G> // G groups of 8 per thread: rows up to 256 x 8 x G samples
__global__ void __launch_bounds__(256)
ozaki_slice_reg_kernel(const double* __restrict__ in, std::size_t ld, std::size_t rows, int K, int nch,
                       int tile_rows, int8_t* __restrict__ sl, int* __restrict__ expo, int* flag) {
    __shared__ double red[8];
    __shared__ int red_bad[8];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const std::size_t r = blockIdx.x;
    const bool real = r < rows;
    const double* row = in + (real ? r * ld : 0);
    const int kend = nch * CB;
    double v[G][8];
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const int k = 8 * t + 2048 * i;
        if (real && k + 8 <= K) {
#pragma unroll
            for (int u = 0; u < 8; u += 2) {
                const double2 a = __ldg(reinterpret_cast<const double2*>(row + k + u));
                v[i][u] = a.x;
                v[i][u + 1] = a.y;
            }
        } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) v[i][u] = (real && k + u < K) ? row[k + u] : 0.0;
        }
    }
    double mx = 0.0;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < G; ++i)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            bad |= !isfinite(v[i][u]);
            mx = fmax(mx, fabs(v[i][u]));
        }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int anybad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
        red[warp] = mx;
        red_bad[warp] = anybad;
    }
    __syncthreads();
    mx = red[0];
    anybad = red_bad[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
        mx = fmax(mx, red[w]);
        anybad |= red_bad[w];
    }
    if (anybad) {
        if (t == 0 && flag) atomicOr(flag, 1);
        mx = 0.0;
    }
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);
    if (t == 0) expo[r] = e;
    const double scale = ldexp(127.0, -e);
    const std::size_t tile = r / tile_rows;
    const int lr = static_cast<int>(r % tile_rows);
    const std::size_t slice_bytes = static_cast<std::size_t>(tile_rows) * CB;
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const int k = 8 * t + 2048 * i;
        if (k >= kend) break;
        double* w = v[i];
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = isfinite(w[u]) ? w[u] * scale : 0.0;
        int8_t* dst = sl + ((tile * nch + k / CB) * S) * slice_bytes + sw64(lr, (k % CB) / 16) + (k % 16);
#pragma unroll
        for (int q = 0; q < S; ++q) {
            uint32_t lo = 0u, hi = 0u;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                lo |= ozaki_digit(w[u]) << (8 * u);
                hi |= ozaki_digit(w[4 + u]) << (8 * u);
            }
            *reinterpret_cast<uint2*>(dst + q * slice_bytes) = make_uint2(lo, hi);
        }
    }
}

/// Folded rows (antisymmetric plans): row r of x (2L samples) becomes the K =
/// 2L operand [y | u], y_j = x_j + x_{2L-1-j}, u_j = x_j - x_{2L-1-j} (j < L),
/// sliced with one exponent per row (max over both halves) — the A side of
/// the grouped product that gives the even (D y) and odd (W u) coefficients
/// of the row in one launch.  A warp per row, 8 rows per CTA; lane l takes 4
/// consecutive j per step (16-byte loads of x_j.. and of the mirrored x).
template <int S, int kMaxSteps> // L <= 128 kMaxSteps
__global__ void __launch_bounds__(256)
ozaki_slice_fold_kernel(const double* __restrict__ in, std::size_t ld, std::size_t rows, std::size_t rows_pad,
                        int L, int tile_rows, int8_t* __restrict__ sl, int* __restrict__ expo, int* flag) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const std::size_t r = static_cast<std::size_t>(blockIdx.x) * 8 + warp;
    if (r >= rows_pad) return;
    const bool real = r < rows;
    const double* row = in + (real ? r * ld : 0);
    const int steps = (L + 127) / 128;
    double y[kMaxSteps][4], u[kMaxSteps][4];
    double mx = 0.0;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < kMaxSteps; ++i) {
        if (i >= steps) break;
        const int j = 4 * lane + 128 * i;
        double a[4] = {0.0, 0.0, 0.0, 0.0}, b[4] = {0.0, 0.0, 0.0, 0.0};
        if (real && j < L) {
            const double2 a0 = __ldg(reinterpret_cast<const double2*>(row + j));
            const double2 a1 = __ldg(reinterpret_cast<const double2*>(row + j + 2));
            const double2 b0 = __ldg(reinterpret_cast<const double2*>(row + 2 * L - 4 - j));
            const double2 b1 = __ldg(reinterpret_cast<const double2*>(row + 2 * L - 2 - j));
            a[0] = a0.x, a[1] = a0.y, a[2] = a1.x, a[3] = a1.y;
            b[0] = b1.y, b[1] = b1.x, b[2] = b0.y, b[3] = b0.x; // x_{2L-1-j-q}
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            bad |= !isfinite(a[q]) || !isfinite(b[q]);
            y[i][q] = a[q] + b[q];
            u[i][q] = a[q] - b[q];
            mx = fmax(mx, fmax(fabs(y[i][q]), fabs(u[i][q])));
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (__any_sync(0xffffffffu, bad)) {
        if (lane == 0 && flag) atomicOr(flag, 1);
        mx = 0.0;
    }
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);
    if (lane == 0) expo[r] = e;
    const double scale = ldexp(127.0, -e);
    const std::size_t tile = r / tile_rows;
    const int lr = static_cast<int>(r % tile_rows), nch = (2 * L + CB - 1) / CB;
    const std::size_t slice_bytes = static_cast<std::size_t>(tile_rows) * CB;
#pragma unroll
    for (int i = 0; i < kMaxSteps; ++i) {
        if (i >= steps) break;
        const int j = 4 * lane + 128 * i;
        if (j >= L) break;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double x = h == 0 ? y[i][q] : u[i][q];
                v[q] = isfinite(x) ? x * scale : 0.0;
            }
            const int k = j + h * L;
            int8_t* dst = sl + ((tile * nch + k / CB) * S) * slice_bytes + sw64(lr, (k % CB) / 16) + (k % 16);
#pragma unroll
            for (int q = 0; q < S; ++q) {
                uint32_t w = 0u;
#pragma unroll
                for (int t = 0; t < 4; ++t) w |= ozaki_digit(v[t]) << (8 * t);
                *reinterpret_cast<uint32_t*>(dst + q * slice_bytes) = w;
            }
        }
    }
}

// ------------------------------------------------------------------- GEMM

template <int S, int NT>
struct Geo {
    static constexpr int kLevels = S;                       // LMAX = S - 1
    static constexpr int kABytes = S * TM * CB;             // A slices of one chunk
    static constexpr int kBBytes = S * NT * CB;             // B slices of one chunk
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStages = (kMaxSmem - 2048) / kStageBytes;
    static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
    static_assert(kLevels * NT <= 512, "TMEM: one NT-column accumulator per level");
    static_assert(kStages >= 2, "at least two pipeline stages");
    static_assert(NT % 16 == 0 && NT >= 16 && NT <= 256, "M = 128 needs N % 16 == 0");
};

/// 2^e as a double for the small exponents of the slicing (|e| < 1000),
/// built from its bit pattern (ldexp's range handling costs ~20 branchy
/// instructions per element in the epilogue).
__device__ __forceinline__ double pow2i(int e) {
    return __longlong_as_double(static_cast<long long>(1023 + e) << 52);
}

/// Epilogue of one 128 x NT tile (rows row0..row0+127, columns nt NT..):
/// warp w reads TMEM lanes 32 w .. 32 w + 31 level by level (Horner in fp64,
/// exact int32 -> fp64 conversions); the 32 x 32 blocks then turn around in
/// shared memory (`stage`: this warp's 32 x 33 doubles) so that every store —
/// plain rows, scattered slots (col_map) or the unfolded pair (fold_add) — is
/// a warp-wide run of consecutive columns of one row (coalesced, whole
/// sectors) instead of 32 rows at once.  Scales: 2^e_b / 127^2 per row before
/// the turn-around, 2^f_c per column (one per lane) after it.  `lsum`
/// (split-K tiles): the level sums come from the tile's accumulated int32
/// sums in global memory ([level * NT + column][lane], red_tile) instead of
/// TMEM — exact integers, so the result is bit-identical to the unsplit tile's.
template <int LEVELS, int NT, bool LSUM = false>
__device__ __forceinline__ void store_tile(uint32_t tmem, std::size_t row0, int nt, int warp, int lane, std::size_t M,
                                           int N, const int* __restrict__ ea, const int* __restrict__ eb,
                                           double* __restrict__ out, std::size_t ld_out,
                                           const int* __restrict__ col_map, const double* __restrict__ fold_add,
                                           std::size_t ld_add, double* stage, const int* lsum = nullptr) {
    constexpr int LDS = 33;
    const std::size_t wrow0 = row0 + 32 * warp, row = wrow0 + lane;
    const double rs = row < M ? pow2i(ea[row]) * (1.0 / (127.0 * 127.0)) : 0.0;
    const int live_rows = wrow0 >= M ? 0 : (M - wrow0 >= 32 ? 32 : static_cast<int>(M - wrow0));
    constexpr double kInv = 1.0 / 254.0;
    const int lim = min(N, nt * NT + NT); // columns of this tile
#pragma unroll 1
    for (int c0 = 0; c0 < NT; c0 += 32) {
        const int cbase = nt * NT + c0;
        if (cbase >= lim) break; // padded column tiles
        if constexpr (LSUM) {
            double acc[32];
            uint32_t v[32];
#pragma unroll 1
            for (int L = LEVELS - 1; L >= 0; --L) {
                const int* src = lsum + static_cast<std::size_t>(L * NT + c0) * 32 + lane;
#pragma unroll
                for (int u = 0; u < 32; ++u) v[u] = c0 + u < NT ? static_cast<uint32_t>(__ldcg(src + u * 32)) : 0u;
                if (L == LEVELS - 1) {
#pragma unroll
                    for (int u = 0; u < 32; ++u) acc[u] = i32_to_f64(v[u]);
                } else {
#pragma unroll
                    for (int u = 0; u < 32; ++u) acc[u] = fma(acc[u], kInv, i32_to_f64(v[u]));
                }
            }
#pragma unroll
            for (int u = 0; u < 32; ++u) stage[lane * LDS + u] = acc[u] * rs;
        } else {
            // 16-column halves: every level's TMEM load in flight before one wait
#pragma unroll 1
            for (int h = 0; h < 32; h += 16) {
                uint32_t v[LEVELS][16];
#pragma unroll
                for (int L = 0; L < LEVELS; ++L)
                    tmem_ld16(tmem + (static_cast<uint32_t>(32 * warp) << 16) + static_cast<uint32_t>(L * NT + c0 + h),
                              v[L]);
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    double a = i32_to_f64(v[LEVELS - 1][u]);
#pragma unroll
                    for (int L = LEVELS - 2; L >= 0; --L) a = fma(a, kInv, i32_to_f64(v[L][u]));
                    stage[lane * LDS + h + u] = a * rs;
                }
            }
        }
        __syncwarp();
        // lane l now carries column c = cbase + l of each of the warp's rows
        const int c = cbase + lane;
        const bool col_ok = c < lim;
        const double cs = col_ok ? pow2i(__ldg(eb + c)) : 0.0;
        const int dst = col_ok ? (col_map ? __ldg(col_map + c) : c) : 0;
        if (col_ok) {
            if (fold_add) { // unfold: x_c = w_c + v_c, x_{2N-1-c} = w_c - v_c; all w loads in flight first
                double wv[32];
#pragma unroll
                for (int r = 0; r < 32; ++r) wv[r] = r < live_rows ? __ldg(fold_add + (wrow0 + r) * ld_add + c) : 0.0;
#pragma unroll
                for (int r = 0; r < 32; ++r)
                    if (r < live_rows) {
                        const double val = stage[r * LDS + lane] * cs;
                        double* orow = out + (wrow0 + r) * ld_out;
                        orow[c] = wv[r] + val;
                        orow[2 * N - 1 - c] = wv[r] - val;
                    }
            } else if (live_rows == 32) {
                double* o = out + wrow0 * ld_out + dst;
#pragma unroll 8
                for (int r = 0; r < 32; ++r) o[r * ld_out] = stage[r * LDS + lane] * cs;
            } else {
                for (int r = 0; r < live_rows; ++r) out[(wrow0 + r) * ld_out + dst] = stage[r * LDS + lane] * cs;
            }
        }
        __syncwarp();
    }
}

/// Split-K tiles (SplitSched): a unit's level sums, warp w's 32 TMEM lanes,
/// added into the tile's int32 accumulator in global memory, [level * NT +
/// column][lane] (16-column TMEM loads; each reduction a 128-byte warp run;
/// fire-and-forget, exact).
template <int LEVELS, int NT>
__device__ __forceinline__ void red_tile(uint32_t tmem, int warp, int lane, int* __restrict__ acc) {
#pragma unroll 1
    for (int L = 0; L < LEVELS; ++L)
#pragma unroll 1
        for (int c0 = 0; c0 < NT; c0 += 16) {
            uint32_t v[16];
            tmem_ld16(tmem + (static_cast<uint32_t>(32 * warp) << 16) + static_cast<uint32_t>(L * NT + c0), v);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            int* d = acc + static_cast<std::size_t>(L * NT + c0) * 32 + lane;
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (c0 + u < NT) atomicAdd(d + u * 32, static_cast<int>(v[u]));
        }
}

/// Split-K tiles: the units of a tile run in any order on any pairs; each
/// adds its level sums (red_tile), then counts in on the tile's counter (one
/// per CTA half and epilogue warp); the last to arrive finishes the tile from
/// the accumulated sums and rearms the counter.  Integer sums: the result is
/// bit-identical to the unsplit tile's.
struct SplitSched {
    std::size_t full = 0;   // whole-tile units (the first `full` tiles)
    int rem = 0;            // tiles split along K (the last rem tiles)
    int nsplit = 1;         // units per split tile
    int* cnt = nullptr;     // per tile, CTA half and epilogue warp: arrival counters (zero at launch)
    int* acc = nullptr;     // ... and that warp's int32 level sums (zero at launch)
    int debug = 0;          // persistent kernel, development knob DCTP_OZAKI_PDEBUG (phase isolation)
    // grouped product: column tiles < nt_split take K chunks [0, kch_split),
    // the others [kch_split, nch) (the folded row's y and u halves); -1: off
    int nt_split = -1, kch_split = 0;
};

/// Work unit u -> (column tile, pair, chunk range, split slot): whole tiles
/// first, then the split tiles' K ranges.
struct Unit {
    std::size_t pair;
    int nt, kb, ke, slot;
};
__device__ __forceinline__ Unit unit_of(std::size_t u, const SplitSched& s, int nch, int ntn, int nfast,
                                        std::size_t npairs) {
    Unit w;
    std::size_t t = u;
    w.kb = 0;
    w.ke = nch;
    w.slot = -1;
    if (u >= s.full) {
        const std::size_t v = u - s.full;
        const int split = static_cast<int>(v / s.rem);
        w.slot = static_cast<int>(v % s.rem);
        t = s.full + w.slot;
        w.kb = static_cast<int>(static_cast<long long>(split) * nch / s.nsplit);
        w.ke = static_cast<int>(static_cast<long long>(split + 1) * nch / s.nsplit);
    }
    if (nfast) {
        w.nt = static_cast<int>(t % ntn);
        w.pair = t / ntn;
    } else {
        w.pair = t % npairs;
        w.nt = static_cast<int>(t / npairs);
    }
    if (s.nt_split >= 0) { // grouped product (never split along K)
        w.kb = w.nt < s.nt_split ? 0 : s.kch_split;
        w.ke = w.nt < s.nt_split ? s.kch_split : nch;
    }
    return w;
}

/// Epilogue of a split unit by one epilogue warp (ew: its TMEM lane quarter);
/// `release` runs once the accumulator has been read.
template <int LEVELS, int NT, class R>
__device__ __forceinline__ void finish_split(const SplitSched& s, const Unit& w, uint32_t rank, uint32_t tmem, int ew,
                                             int lane, std::size_t M, int N, const int* ea, const int* eb, double* out,
                                             std::size_t ld_out, const int* col_map, const double* fold_add,
                                             std::size_t ld_add, double* stage, R&& release) {
    const std::size_t blk = (static_cast<std::size_t>(w.slot) * 2 + rank) * 4 + ew;
    int* acc = s.acc + blk * (static_cast<std::size_t>(LEVELS) * NT * 32);
    red_tile<LEVELS, NT>(tmem, ew, lane, acc);
    release();
    __threadfence();
    __syncwarp();
    int old = 0;
    if (lane == 0) old = atomicAdd(s.cnt + blk, 1);
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old == s.nsplit - 1) {
        __threadfence();
        store_tile<LEVELS, NT, true>(tmem, (2 * w.pair + rank) * TM, w.nt, ew, lane, M, N, ea, eb, out, ld_out,
                                     col_map, fold_add, ld_add, stage, acc);
        if (lane == 0) s.cnt[blk] = 0;
    }
}

/// Split of the tail: nsplit minimising the tail's length in waves,
/// ceil(rem * nsplit / slots) / nsplit, plus 3% of a wave per extra split
/// and 30% for splitting at all (measured on C5's shapes: the units' own
/// pipeline fill, the reductions and the finishing epilogue); every unit
/// keeps >= 8 chunks.  DCTP_OZAKI_SPLIT = 0 turns it off; by default
/// products with K >= 2048.
static void plan_split(std::size_t tiles, std::size_t slots, int nch, SplitSched& s) {
    static const int knob = [] {
        const char* e = std::getenv("DCTP_OZAKI_SPLIT");
        return e ? std::atoi(e) : -1;
    }();
    s.full = tiles;
    s.rem = 0;
    s.nsplit = 1;
    const std::size_t rem = tiles % slots;
    if (knob == 0 || rem == 0 || (knob < 0 && nch < 32)) return;
    double best = 1.0;
    int bn = 1;
    for (int ns = 2; ns <= 16 && nch / ns >= 8; ++ns) {
        const double w = static_cast<double>((rem * ns + slots - 1) / slots) / ns + 0.03 * (ns - 1) + 0.3;
        if (w < best - 1e-9) {
            best = w;
            bn = ns;
        }
    }
    if (bn == 1) return;
    s.full = tiles - rem;
    s.rem = static_cast<int>(rem);
    s.nsplit = bn;
}

/// Stream-ordered split workspace (counters + accumulators, zeroed); freed by
/// split_free after the launch.
static cudaError_t split_alloc(SplitSched& s, std::size_t ints_per_blk, cudaStream_t stream, void** ws,
                               int blocks_per_tile = 8) {
    *ws = nullptr;
    if (s.rem == 0) return cudaSuccess;
    const std::size_t nblk = static_cast<std::size_t>(s.rem) * blocks_per_tile;
    const std::size_t cnt_bytes = (nblk * sizeof(int) + 255) / 256 * 256;
    const std::size_t bytes = cnt_bytes + nblk * ints_per_blk * sizeof(int);
    cudaError_t e = cudaMallocAsync(ws, bytes, stream);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(*ws, 0, bytes, stream);
    s.cnt = static_cast<int*>(*ws);
    s.acc = reinterpret_cast<int*>(static_cast<char*>(*ws) + cnt_bytes);
    return e;
}

template <int S, int NT>
__global__ void __launch_bounds__(kThreads, 1)
ozaki_gemm_kernel(const int8_t* __restrict__ a_sl, const int* __restrict__ ea, const int8_t* __restrict__ b_sl,
                  const int* __restrict__ eb, std::size_t M, int N, int nch, double* __restrict__ out,
                  std::size_t ld_out, const int* __restrict__ col_map, const double* __restrict__ fold_add,
                  std::size_t ld_add, int debug) {
    using G = Geo<S, NT>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t raw = ptx::smem_addr(smem_raw);
    unsigned char* base = smem_raw + ((1024 - (raw & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + G::kStages * G::kStageBytes);
    uint64_t* empty = full + G::kStages;
    uint64_t* done = empty + G::kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    const uint32_t sbase = ptx::smem_addr(base);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // grid x = row tile (fastest): the CTAs in flight share their B column tile
    const std::size_t mt = blockIdx.x;
    const int nt = blockIdx.y;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                         ptx::smem_addr(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    if (tid == 32) {
        for (int i = 0; i < G::kStages; ++i) {
            ptx::mbar_init(full + i, 1);
            ptx::mbar_init(empty + i, 1);
        }
        ptx::mbar_init(done, 1);
        ptx::fence_mbar_init();
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    const int8_t* a_tile = a_sl + mt * static_cast<std::size_t>(nch) * G::kABytes;
    const int8_t* b_tile = b_sl + static_cast<std::size_t>(nt) * nch * G::kBBytes;

    if (warp == 0) { // producer warp: one A and one B bulk copy per chunk
        // development knob DCTP_OZAKI_DEBUG=1: load only the first ring of
        // chunks (the MMAs then reuse them: tensor-pipe time alone)
        const int nload = (debug & 1) ? (nch < G::kStages ? nch : G::kStages) : nch;
        for (int ch = 0; ch < nload; ++ch) {
            const int st = ch % G::kStages;
            if (ch >= G::kStages) ptx::mbar_wait(empty + st, static_cast<uint32_t>(((ch / G::kStages) - 1) & 1));
            if (elect_one()) {
                ptx::mbar_expect_tx(full + st, G::kStageBytes);
                unsigned char* dst = base + st * G::kStageBytes;
                ptx::bulk_load(dst, a_tile + static_cast<std::size_t>(ch) * G::kABytes, G::kABytes, full + st);
                ptx::bulk_load(dst + G::kABytes, b_tile + static_cast<std::size_t>(ch) * G::kBBytes, G::kBBytes,
                               full + st);
            }
            __syncwarp();
        }
    } else if (warp == 1) { // MMA warp: one elected lane issues, the warp stays converged
        // descriptors of stage 0; other stages / slices / K steps add their
        // byte offset / 16 to the 14-bit start-address field (< 256 KB: no carry)
        const uint64_t adesc0 = smem_desc(sbase), bdesc0 = smem_desc(sbase + G::kABytes);
        for (int ch = 0; ch < nch; ++ch) {
            const int st = ch % G::kStages;
            if (!(debug & 1) || ch < G::kStages) ptx::mbar_wait(full + st, static_cast<uint32_t>((ch / G::kStages) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            if (elect_one()) {
                const uint64_t so = static_cast<uint64_t>(st * G::kStageBytes) >> 4;
                const uint64_t ad = adesc0 + so, bd = bdesc0 + so;
                // slice i outer, j inner: consecutive MMAs write different
                // level accumulators (L = i + j), never the one just issued
#pragma unroll
                for (int kk = 0; kk < CB / 32; ++kk) {
#pragma unroll
                    for (int i = 0; i < G::kLevels; ++i) {
#pragma unroll
                        for (int j = 0; i + j < G::kLevels; ++j) {
                            const int L = i + j;
                            const uint32_t td = tmem + static_cast<uint32_t>(L * NT);
                            const uint32_t acc = (ch > 0 || kk > 0 || i > 0) ? 1u : 0u;
                            if (!(debug & 2)) // DCTP_OZAKI_DEBUG=2: loads only
                                mma_i8<NT>(td, ad + ((i * TM * CB + 32 * kk) >> 4), bd + ((j * NT * CB + 32 * kk) >> 4),
                                           acc);
                        }
                    }
                }
                mma_commit(empty + st);
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(done);
        __syncwarp();
    }

    // epilogue: warp w reads TMEM lanes 32 w .. 32 w + 31 (tile rows)
    ptx::mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    store_tile<G::kLevels, NT>(tmem, mt * TM, nt, warp, lane, M, N, ea, eb, out, ld_out, col_map, fold_add, ld_add,
                               reinterpret_cast<double*>(base) + warp * 32 * 33);
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
}

// ---------------------------------------------------------- CTA-pair GEMM

/// Geometry of the CTA-pair kernel: an MMA is M = 256 (128 rows per CTA) x
/// N = NT; each CTA stages its own 128 A rows and one half (NT / 2 rows) of
/// the B tile, so per SM the tensor core reads 128 + NT/2 operand rows per
/// K step instead of 128 + NT (the shared-memory read rate is what holds the
/// single-CTA N = 96 MMA at ~82% of the tensor peak).
template <int S, int NT>
struct Geo2 {
    static constexpr int kLevels = S;
    static constexpr int kHalf = NT / 2;
    static constexpr int kABytes = S * TM * CB;
    static constexpr int kBBytes = S * kHalf * CB;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStages = (kMaxSmem - 2048) / kStageBytes;
    static constexpr int kSmem = kStages * kStageBytes + 1024 + 512;
    static_assert(kLevels * NT <= 512, "TMEM: one NT-column accumulator per level");
    static_assert(kStages >= 2, "at least two pipeline stages");
    static_assert(NT % 16 == 0 && NT <= 256 && kHalf % 8 == 0,
                  "cta_group::2 with M = 256 needs N % 16 == 0; each half whole 8-row swizzle groups");
};

template <int NT>
__host__ __device__ constexpr uint32_t idesc_i8_pair() {
    return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(NT >> 3) << 17) |
           (static_cast<uint32_t>(256 >> 4) << 24);
}

template <int NT>
__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc_i8_pair<NT>()), "r"(accumulate));
}

/// Commit of the pair's MMAs, arriving on the barrier at the same offset in
/// every CTA of `mask`.
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            ptx::smem_addr(bar)),
        "h"(mask)
        : "memory");
}

/// 1-D bulk copy global -> the same shared offset in every CTA of `mask`,
/// completing on each destination's mbarrier at `bar`'s offset.
__device__ __forceinline__ void bulk_load_mcast(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
        "%4;\n" ::"r"(ptx::smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(ptx::smem_addr(bar)), "h"(mask)
        : "memory");
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

/// Arrive on the mbarrier at `bar`'s offset in CTA `rank` of the cluster.
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
    asm volatile(
        "{\n.reg .b32 ra;\nmapa.shared::cluster.u32 ra, %0, %1;\n"
        "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}\n" ::"r"(ptx::smem_addr(bar)),
        "r"(rank)
        : "memory");
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAITC_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITC_%=;\n}\n" ::"r"(ptx::smem_addr(bar)),
        "r"(parity)
        : "memory");
}

/// Clusters of 2 x NSUB CTAs: NSUB CTA pairs along N, each pair two CTAs
/// along M.  In a pair, the CTA with M-half h holds rows 128 h.. of the
/// pair's 256-row tile and B rows (NT / 2) h.. of the pair's column tile (B
/// sliced with tile_rows = NT / 2, so its half is tile 2 nt + h).  The h = 0
/// CTA issues the cta_group::2 MMAs once both CTAs' stage landed: the h = 1
/// CTA's warp 2 relays its full barrier to the leader's peer_full barrier.
/// Each CTA's TMEM holds its 128 rows of every level accumulator and runs its
/// own epilogue.  NSUB = 2: the two pairs share the same 256 rows, so each CTA
/// loads one half of its A chunk and multicasts it to its counterpart in the
/// other pair — A's L2 reads halve (the operand traffic, not the MMAs, held
/// the pair kernel at ~67% of the tensor pipe); both leaders' commits then
/// arrive on every CTA's empty barrier.
template <int S, int NT, int NSUB>
__global__ void __launch_bounds__(kThreads, 1)
ozaki_gemm2_kernel(const int8_t* __restrict__ a_sl, const int* __restrict__ ea, const int8_t* __restrict__ b_sl,
                   const int* __restrict__ eb, std::size_t M, int N, int nch, double* __restrict__ out,
                   std::size_t ld_out, const int* __restrict__ col_map, const double* __restrict__ fold_add,
                   std::size_t ld_add, int ntn, int nfast, std::size_t npairs, int debug, SplitSched sched) {
    using G = Geo2<S, NT>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t raw = ptx::smem_addr(smem_raw);
    unsigned char* base = smem_raw + ((1024 - (raw & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + G::kStages * G::kStageBytes);
    uint64_t* peer_full = full + G::kStages;
    uint64_t* empty = peer_full + G::kStages;
    uint64_t* done = empty + G::kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    const uint32_t sbase = ptx::smem_addr(base);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint32_t q = 0;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(q));
    const uint32_t rank = q & 1u, ns = q >> 1; // M half within the pair, pair index
    // this CTA's 128-row tile (pairs: 2 p, 2 p + 1) and column tile.  nfast:
    // consecutive clusters walk the column tiles of one row pair (the B
    // operand stays in L2 and A streams once: short-K products such as the
    // chain); otherwise row pairs fastest (B, the larger operand, streams once)
    std::size_t mt;
    int nt;
    Unit w{0, 0, 0, nch, -1}; // split-K tail (NSUB = 1): whole tiles, then K ranges of the last tiles
    if (NSUB == 1 && sched.rem > 0) {
        w = unit_of(blockIdx.x / 2, sched, nch, ntn, nfast, npairs);
        mt = 2 * w.pair + rank;
        nt = w.nt;
    } else if (NSUB == 1 && !nfast) {
        mt = blockIdx.x;
        nt = blockIdx.y;
    } else {
        const std::size_t ci = blockIdx.x / (2 * NSUB);
        const std::size_t ntc = (static_cast<std::size_t>(ntn) + NSUB - 1) / NSUB; // column-tile groups
        std::size_t p, g;
        if (nfast) {
            g = ci % ntc;
            p = ci / ntc;
        } else {
            p = ci % npairs;
            g = ci / npairs;
        }
        nt = static_cast<int>(g * NSUB + ns);
        mt = 2 * p + rank;
    }

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                         ptx::smem_addr(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
    }
    if (tid == 32) {
        for (int i = 0; i < G::kStages; ++i) {
            ptx::mbar_init(full + i, 1);
            ptx::mbar_init(peer_full + i, 1);
            ptx::mbar_init(empty + i, NSUB); // one commit from each pair's leader
        }
        ptx::mbar_init(done, 1);
        ptx::fence_mbar_init();
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    cluster_sync(); // every CTA's barriers and TMEM exist before any cross-CTA traffic
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    const int8_t* a_tile = a_sl + (mt * static_cast<std::size_t>(nch) + w.kb) * G::kABytes;
    const int8_t* b_tile = b_sl + ((2 * static_cast<std::size_t>(nt) + rank) * nch + w.kb) * G::kBBytes;
    nch = w.ke - w.kb; // this unit's chunks

    const uint16_t all_mask = static_cast<uint16_t>((1u << (2 * NSUB)) - 1u);
    const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2 * ns));
    // development knob DCTP_OZAKI_DEBUG=1: only the first ring of chunks is
    // loaded (the MMAs reuse it: tensor-pipe time alone)
    const int nload = (debug & 1) ? (nch < G::kStages ? nch : G::kStages) : nch;
    if (warp == 0) { // producer warp (every CTA): this CTA's A rows and B half
        for (int ch = 0; ch < nload; ++ch) {
            const int st = ch % G::kStages;
            if (ch >= G::kStages) ptx::mbar_wait(empty + st, static_cast<uint32_t>(((ch / G::kStages) - 1) & 1));
            if (elect_one()) {
                ptx::mbar_expect_tx(full + st, G::kStageBytes);
                unsigned char* dst = base + st * G::kStageBytes;
                const int8_t* asrc = a_tile + static_cast<std::size_t>(ch) * G::kABytes;
                if constexpr (NSUB == 2) { // half of the A chunk, to this CTA and its counterpart
                    constexpr uint32_t half = G::kABytes / 2;
                    bulk_load_mcast(dst + ns * half, asrc + ns * half, half, full + st,
                                    static_cast<uint16_t>((1u << q) | (1u << (q ^ 2u))));
                } else {
                    ptx::bulk_load(dst, asrc, G::kABytes, full + st);
                }
                ptx::bulk_load(dst + G::kABytes, b_tile + static_cast<std::size_t>(ch) * G::kBBytes, G::kBBytes,
                               full + st);
            }
            __syncwarp();
        }
    } else if (warp == 1 && rank == 0) { // MMA warp of the pair
        const uint64_t adesc0 = smem_desc(sbase), bdesc0 = smem_desc(sbase + G::kABytes);
        for (int ch = 0; ch < nch; ++ch) {
            const int st = ch % G::kStages;
            const uint32_t ph = static_cast<uint32_t>((ch / G::kStages) & 1);
            if (ch < nload) {
                ptx::mbar_wait(full + st, ph);
                mbar_wait_cluster(peer_full + st, ph);
            }
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            if (elect_one()) {
                const uint64_t so = static_cast<uint64_t>(st * G::kStageBytes) >> 4;
                const uint64_t ad = adesc0 + so, bd = bdesc0 + so;
#pragma unroll
                for (int kk = 0; kk < CB / 32; ++kk) {
#pragma unroll
                    for (int i = 0; i < G::kLevels; ++i) {
#pragma unroll
                        for (int j = 0; i + j < G::kLevels; ++j) {
                            const uint32_t td = tmem + static_cast<uint32_t>((i + j) * NT);
                            const uint32_t acc = (ch > 0 || kk > 0 || i > 0) ? 1u : 0u;
                            mma_i8_pair<NT>(td, ad + ((i * TM * CB + 32 * kk) >> 4),
                                            bd + ((j * G::kHalf * CB + 32 * kk) >> 4), acc);
                        }
                    }
                }
                mma_commit_pair(empty + st, all_mask);
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit_pair(done, pair_mask);
        __syncwarp();
    } else if (warp == 2 && rank == 1) { // relay: this CTA's stage landed -> the pair's leader
        for (int ch = 0; ch < nload; ++ch) {
            const int st = ch % G::kStages;
            ptx::mbar_wait(full + st, static_cast<uint32_t>((ch / G::kStages) & 1));
            if (elect_one()) mbar_arrive_remote(peer_full + st, q - 1);
            __syncwarp();
        }
    }

    ptx::mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (w.slot >= 0)
        finish_split<G::kLevels, NT>(sched, w, rank, tmem, warp, lane, M, N, ea, eb, out, ld_out, col_map, fold_add,
                                     ld_add, reinterpret_cast<double*>(base) + warp * 32 * 33, [] {});
    else if (!(debug & 4)) // DCTP_OZAKI_DEBUG=4: no epilogue (timing only)
        store_tile<G::kLevels, NT>(tmem, mt * TM, nt, warp, lane, M, N, ea, eb, out, ld_out, col_map, fold_add,
                                   ld_add, reinterpret_cast<double*>(base) + warp * 32 * 33);
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    cluster_sync(); // no peer traffic into this CTA is still pending
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
}

// ------------------------------------------------------ persistent CTA pairs

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}

/// Persistent-kernel epilogue, phase 1 (accumulator -> registers): the warp
/// with TMEM lane quarter q and column half h reads its 32 rows x NT/2
/// columns, every level of an 8-column group in flight before one wait,
/// Horner in fp64 (exact int32 -> fp64) and the row scale 2^e_b / 127^2.  The
/// accumulator is free for the next unit's MMAs as soon as every epilogue
/// warp has done this — the stores (phase 2) then overlap those MMAs.
template <int LEVELS, int NT>
__device__ __forceinline__ void drain_half(uint32_t tmem, int q, int h, double rs, double (&acc)[NT / 2]) {
    constexpr int H = NT / 2;
    constexpr double kInv = 1.0 / 254.0;
#pragma unroll
    for (int g = 0; g < H; g += 8) {
        uint32_t v[LEVELS][8];
#pragma unroll
        for (int L = 0; L < LEVELS; ++L)
            tmem_ld8(tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(L * NT + h * H + g), v[L]);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            double a = i32_to_f64(v[LEVELS - 1][u]);
#pragma unroll
            for (int L = LEVELS - 2; L >= 0; --L) a = fma(a, kInv, i32_to_f64(v[L][u]));
            acc[g + u] = a * rs;
        }
    }
}

/// Split-K units, phase 1: the same 32 x NT/2 block from the tile's summed
/// int32 levels in global memory ([level][column][lane], exact), so a split
/// tile ends bit-identical to an unsplit one.
template <int LEVELS, int NT>
__device__ __forceinline__ void drain_half_sum(const int* __restrict__ lsum, int lane, double rs,
                                               double (&acc)[NT / 2]) {
    constexpr int H = NT / 2;
    constexpr double kInv = 1.0 / 254.0;
#pragma unroll
    for (int u = 0; u < H; ++u)
        acc[u] = i32_to_f64(static_cast<uint32_t>(__ldcg(lsum + static_cast<std::size_t>((LEVELS - 1) * H + u) * 32 + lane)));
#pragma unroll 1
    for (int L = LEVELS - 2; L >= 0; --L)
#pragma unroll
        for (int u = 0; u < H; ++u)
            acc[u] = fma(acc[u], kInv,
                         i32_to_f64(static_cast<uint32_t>(__ldcg(lsum + static_cast<std::size_t>(L * H + u) * 32 + lane))));
#pragma unroll
    for (int u = 0; u < H; ++u) acc[u] *= rs;
}

/// Split-K units: this warp's level sums added into the tile's int32
/// accumulator ([level][column][lane], 128-byte warp runs, fire-and-forget).
template <int LEVELS, int NT>
__device__ __forceinline__ void red_half(uint32_t tmem, int q, int h, int lane, int* __restrict__ acc) {
    constexpr int H = NT / 2;
#pragma unroll 1
    for (int L = 0; L < LEVELS; ++L)
#pragma unroll
        for (int g = 0; g < H; g += 8) {
            uint32_t v[8];
            tmem_ld8(tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(L * NT + h * H + g), v);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            int* d = acc + static_cast<std::size_t>(L * H + g) * 32 + lane;
#pragma unroll
            for (int u = 0; u < 8; ++u) atomicAdd(d + u * 32, static_cast<int>(v[u]));
        }
}

/// Column constants of one warp's half tile, per lane (j = lane & 15) and
/// 16-column block: the column scale 2^f_c and the destination column —
/// loaded before the accumulator is ready, so the stores wait on nothing.
template <int NT>
struct HalfCols {
    static constexpr int kBlocks = (NT / 2 + 15) / 16;
    double cs[kBlocks];
    int dst[kBlocks];
    __device__ __forceinline__ void load(int c0, int lane, int N, const int* __restrict__ eb,
                                         const int* __restrict__ col_map) {
        constexpr int H = NT / 2;
        const int j = lane & 15;
#pragma unroll
        for (int k = 0; k < kBlocks; ++k) {
            const int b = 16 * k, c = c0 + b + j;
            const bool ok = b + j < H && c < N;
            cs[k] = ok ? pow2i(__ldg(eb + c)) : 0.0;
            dst[k] = ok ? (col_map ? __ldg(col_map + c) : c) : -1;
        }
    }
};

/// Persistent-kernel epilogue, phase 2 (registers -> HBM): 16-column blocks
/// of the warp's 32 x NT/2 values turn around in shared memory (32 x 17
/// doubles) so that each store instruction writes two rows x 16 consecutive
/// columns (whole 128-byte lines for plain rows); lane (j, r&1) then applies
/// the column scale 2^f_c and writes plain rows, scattered slots (col_map) or
/// the unfolded pair (fold_add: x_c = w_c + v_c, x_{2N-1-c} = w_c - v_c).
template <int NT>
__device__ __forceinline__ void store_half(const double (&acc)[NT / 2], const HalfCols<NT>& hc, std::size_t wrow0,
                                           int c0, int lane, std::size_t M, int N, double* __restrict__ out,
                                           std::size_t ld_out, const double* __restrict__ fold_add, std::size_t ld_add,
                                           double* stage) {
    constexpr int H = NT / 2, LDS = 17;
    const int live_rows = wrow0 >= M ? 0 : (M - wrow0 >= 32 ? 32 : static_cast<int>(M - wrow0));
    const int j = lane & 15, rp = lane >> 4;
#pragma unroll
    for (int k = 0; k < HalfCols<NT>::kBlocks; ++k) {
        const int b = 16 * k;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (b + u < H) stage[lane * LDS + u] = acc[b + u];
        __syncwarp();
        const double cs = hc.cs[k];
        const int dst = hc.dst[k];
        if (dst >= 0) {
            if (fold_add) {
                const int c = c0 + b + j;
                double wv[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int r = 2 * i + rp;
                    wv[i] = r < live_rows ? __ldg(fold_add + (wrow0 + r) * ld_add + c) : 0.0;
                }
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int r = 2 * i + rp;
                    if (r < live_rows) {
                        const double val = stage[r * LDS + j] * cs;
                        double* orow = out + (wrow0 + r) * ld_out;
                        orow[c] = wv[i] + val;
                        orow[2 * N - 1 - c] = wv[i] - val;
                    }
                }
            } else {
                double* o = out + (wrow0 + rp) * ld_out + dst;
                if (live_rows == 32) {
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        __stcs(o + 2 * i * ld_out, stage[(2 * i + rp) * LDS + j] * cs);
                } else {
                    for (int i = 0; 2 * i + rp < live_rows; ++i)
                        __stcs(o + 2 * i * ld_out, stage[(2 * i + rp) * LDS + j] * cs);
                }
            }
        }
        __syncwarp();
    }
}

/// Geometry of the persistent pair kernel: a 3-stage ring (the epilogue needs
/// its own staging: the ring keeps loading the next tile meanwhile).
template <int S, int NT>
struct GeoP {
    static constexpr int kLevels = S;
    static constexpr int kHalf = NT / 2;
    static constexpr int kABytes = S * TM * CB;
    static constexpr int kBBytes = S * kHalf * CB;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStaging = 8 * 32 * 17 * 8; // 8 epilogue warps x 32 x 17 doubles
    static constexpr int kStages = (kMaxSmem - 2048 - kStaging) / kStageBytes;
    static constexpr int kSmem = kStages * kStageBytes + kStaging + 1024 + 512;
    static_assert(kLevels * NT <= 512, "TMEM: one NT-column accumulator per level");
    static_assert(kStages >= 2, "at least two pipeline stages");
    static_assert(NT % 16 == 0 && (NT / 2) % 8 == 0, "column halves of whole 8-column groups");
};
// warp 0 producer, 1 MMA (rank 0), 2 relay (rank 1), 4-11 epilogue (lane
// quarter warp % 4, column half (warp - 4) / 4)
constexpr int kPThreads = 384;
constexpr int kPEpiWarps = 8;

/// Persistent CTA pairs (cluster of 2 along M, cta_group::2 MMAs as in
/// ozaki_gemm2_kernel) over work units u = cluster, cluster + clusters, ...:
/// the producer streams the chunks of consecutive units through one ring (the
/// next unit's first stages load while the current unit's MMAs and epilogue
/// run), so the per-tile prologue, pipeline fill and teardown of the one-tile
/// kernel are paid once — what dominates short products (K = 512 .. 2048:
/// the folded products and the rank-k chain).  The accumulator (5 x 96 TMEM
/// columns) is single-buffered, but held only while the epilogue drains it:
/// eight epilogue warps per CTA (lane quarter x column half) copy it into
/// registers (Horner, row scale), release it (t_empty: 16 arrivals at the
/// leader) and only then store, so unit i's stores overlap unit i + 1's MMAs.
///
/// Split-K tail (SplitSched): the first `full` units are whole tiles; the
/// remaining `rem` tiles — a partial last wave — are split along K into
/// `nsplit` units each, so the tail costs ~1/nsplit of a wave instead of a
/// whole one (C5 sharded 8 ways, 256 rows: 86 column tiles on 74 pairs).
template <int S, int NT, bool SPLIT>
__global__ void __launch_bounds__(kPThreads, 1)
ozaki_gemmp_kernel(const int8_t* __restrict__ a_sl, const int* __restrict__ ea, const int8_t* __restrict__ b_sl,
                   const int* __restrict__ eb, std::size_t M, int N, int nch, double* __restrict__ out,
                   std::size_t ld_out, const int* __restrict__ col_map, const double* __restrict__ fold_add,
                   std::size_t ld_add, int ntn, int nfast, std::size_t npairs, SplitSched sched) {
    using G = GeoP<S, NT>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t raw = ptx::smem_addr(smem_raw);
    unsigned char* base = smem_raw + ((1024 - (raw & 1023)) & 1023);
    double* staging = reinterpret_cast<double*>(base + G::kStages * G::kStageBytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + G::kStages * G::kStageBytes + G::kStaging);
    uint64_t* peer_full = full + G::kStages;
    uint64_t* empty = peer_full + G::kStages;
    uint64_t* t_full = empty + G::kStages;  // accumulator complete (leader's commit, both CTAs)
    uint64_t* t_empty = t_full + 1;         // accumulator drained (leader: 4 local + 4 peer epilogue warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + 1);
    const uint32_t sbase = ptx::smem_addr(base);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint32_t rank = 0;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const std::size_t clusters = gridDim.x / 2, cid = blockIdx.x / 2;
    const std::size_t units = sched.full + static_cast<std::size_t>(sched.rem) * sched.nsplit;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                         ptx::smem_addr(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
    }
    if (tid == 32) {
        for (int i = 0; i < G::kStages; ++i) {
            ptx::mbar_init(full + i, 1);
            ptx::mbar_init(peer_full + i, 1);
            ptx::mbar_init(empty + i, 1);
        }
        ptx::mbar_init(t_full, 1);
        ptx::mbar_init(t_empty, 2 * kPEpiWarps);
        ptx::fence_mbar_init();
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) { // producer (both CTAs): chunks of every unit of this pair, one ring
        unsigned long long q = 0;
        for (std::size_t u = cid; u < units; u += clusters) {
            const Unit w = unit_of(u, sched, nch, ntn, nfast, npairs);
            const int8_t* a_tile = a_sl + (2 * w.pair + rank) * static_cast<std::size_t>(nch) * G::kABytes;
            const int8_t* b_tile = b_sl + (2 * static_cast<std::size_t>(w.nt) + rank) * nch * G::kBBytes;
            for (int ch = w.kb; ch < w.ke; ++ch, ++q) {
                const int st = static_cast<int>(q % G::kStages);
                if (q >= static_cast<unsigned long long>(G::kStages))
                    ptx::mbar_wait(empty + st, static_cast<uint32_t>(((q / G::kStages) - 1) & 1));
                if (elect_one()) {
                    ptx::mbar_expect_tx(full + st, G::kStageBytes);
                    unsigned char* dst = base + st * G::kStageBytes;
                    ptx::bulk_load(dst, a_tile + static_cast<std::size_t>(ch) * G::kABytes, G::kABytes, full + st);
                    ptx::bulk_load(dst + G::kABytes, b_tile + static_cast<std::size_t>(ch) * G::kBBytes,
                                   G::kBBytes, full + st);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1 && rank == 0) { // MMA warp of the pair
        const uint64_t adesc0 = smem_desc(sbase), bdesc0 = smem_desc(sbase + G::kABytes);
        unsigned long long q = 0;
        int i = 0;
        for (std::size_t u = cid; u < units; u += clusters, ++i) {
            const Unit w = unit_of(u, sched, nch, ntn, nfast, npairs);
            if (i > 0) mbar_wait_cluster(t_empty, static_cast<uint32_t>((i - 1) & 1)); // epilogues drained TMEM
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            for (int ch = w.kb; ch < w.ke; ++ch, ++q) {
                const int st = static_cast<int>(q % G::kStages);
                const uint32_t ph = static_cast<uint32_t>((q / G::kStages) & 1);
                ptx::mbar_wait(full + st, ph);
                mbar_wait_cluster(peer_full + st, ph);
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                if (elect_one()) {
                    const uint64_t so = static_cast<uint64_t>(st * G::kStageBytes) >> 4;
                    const uint64_t ad = adesc0 + so, bd = bdesc0 + so;
#pragma unroll
                    for (int kk = 0; kk < CB / 32; ++kk) {
#pragma unroll
                        for (int a = 0; a < G::kLevels; ++a) {
#pragma unroll
                            for (int b = 0; a + b < G::kLevels; ++b) {
                                const uint32_t td = tmem + static_cast<uint32_t>((a + b) * NT);
                                const uint32_t acc = (ch > w.kb || kk > 0 || a > 0) ? 1u : 0u;
                                if (!(sched.debug & 8)) // development: loads only
                                    mma_i8_pair<NT>(td, ad + ((a * TM * CB + 32 * kk) >> 4),
                                                    bd + ((b * G::kHalf * CB + 32 * kk) >> 4), acc);
                            }
                        }
                    }
                    mma_commit_pair(empty + st, 0x3);
                }
                __syncwarp();
            }
            if (elect_one()) mma_commit_pair(t_full, 0x3);
            __syncwarp();
        }
    } else if (warp == 2 && rank == 1) { // relay: this CTA's stage landed -> the leader
        unsigned long long q = 0;
        for (std::size_t u = cid; u < units; u += clusters) {
            const Unit w = unit_of(u, sched, nch, ntn, nfast, npairs);
            for (int ch = w.kb; ch < w.ke; ++ch, ++q) {
                const int st = static_cast<int>(q % G::kStages);
                ptx::mbar_wait(full + st, static_cast<uint32_t>((q / G::kStages) & 1));
                if (elect_one()) mbar_arrive_remote(peer_full + st, 0);
                __syncwarp();
            }
        }
    } else if (warp >= 4) { // epilogue warps: TMEM lane quarter warp % 4, column half (warp - 4) / 4
        constexpr int H = NT / 2;
        const int ew = warp - 4, q = warp & 3, h = ew >> 2;
        double* stage = staging + ew * 32 * 17;
        int i = 0;
        auto release = [&] { // every epilogue warp of both CTAs releases the pair's accumulator at the leader
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                if (rank == 0)
                    ptx::mbar_arrive(t_empty);
                else
                    mbar_arrive_remote(t_empty, 0);
            }
        };
        for (std::size_t u = cid; u < units; u += clusters, ++i) {
            const Unit w = unit_of(u, sched, nch, ntn, nfast, npairs);
            const std::size_t wrow0 = (2 * w.pair + rank) * TM + 32 * q, row = wrow0 + lane;
            const double rs = row < M ? pow2i(__ldg(ea + row)) * (1.0 / (127.0 * 127.0)) : 0.0;
            HalfCols<NT> hc;
            hc.load(w.nt * NT + h * H, lane, N, eb, (sched.debug & 4) ? nullptr : col_map);
            ptx::mbar_wait(t_full, static_cast<uint32_t>(i & 1));
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            double acc[H];
            if (!SPLIT || w.slot < 0) {
                if (sched.debug & 2) { // development: no drain
#pragma unroll
                    for (int c = 0; c < H; ++c) acc[c] = rs;
                } else {
                    drain_half<G::kLevels, NT>(tmem, q, h, rs, acc);
                }
                release(); // the next unit's MMAs may start: the stores below overlap them
                if (sched.debug & 1) continue; // development: no stores
            } else {
                const std::size_t blk = (static_cast<std::size_t>(w.slot) * 2 + rank) * kPEpiWarps + ew;
                int* lsum = sched.acc + blk * (static_cast<std::size_t>(G::kLevels) * H * 32);
                red_half<G::kLevels, NT>(tmem, q, h, lane, lsum);
                release();
                __threadfence();
                __syncwarp();
                int old = 0;
                if (lane == 0) old = atomicAdd(sched.cnt + blk, 1);
                old = __shfl_sync(0xffffffffu, old, 0);
                if (old != sched.nsplit - 1) continue; // another unit of this tile finishes it
                __threadfence();
                drain_half_sum<G::kLevels, NT>(lsum, lane, rs, acc);
                if (lane == 0) sched.cnt[blk] = 0;
            }
            store_half<NT>(acc, hc, wrow0, w.nt * NT + h * H, lane, M, N, out, ld_out, fold_add, ld_add, stage);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    cluster_sync();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
}

template <int S, int NT>
cudaError_t launch_gemmp(const int8_t* a_sl, const int* ea, const int8_t* b_sl, const int* eb, std::size_t M, int N,
                         int nch, double* out, std::size_t ld_out, const int* col_map, const double* fold_add,
                         std::size_t ld_add, cudaStream_t stream, int nt_split = -1, int kch_split = 0) {
    using G = GeoP<S, NT>;
    cudaError_t e = smem_optin(reinterpret_cast<const void*>(ozaki_gemmp_kernel<S, NT, false>), G::kSmem);
    if (e == cudaSuccess) e = smem_optin(reinterpret_cast<const void*>(ozaki_gemmp_kernel<S, NT, true>), G::kSmem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const std::size_t npairs = (M + 2 * TM - 1) / (2 * TM);
    const int ntn = (N + NT - 1) / NT;
    const std::size_t a_bytes = npairs * 2 * TM * static_cast<std::size_t>(nch) * CB * S;
    const std::size_t b_bytes = static_cast<std::size_t>(ntn) * NT * nch * CB * S;
    const int nfast = b_bytes < a_bytes ? 1 : 0;
    const std::size_t tiles = npairs * ntn;
    SplitSched sched;
    if (nt_split < 0) {
        plan_split(tiles, static_cast<std::size_t>(sms / 2), nch, sched);
    } else {
        sched.full = tiles;
        sched.nt_split = nt_split;
        sched.kch_split = kch_split;
    }
    static const int pdebug = [] {
        const char* v = std::getenv("DCTP_OZAKI_PDEBUG");
        return v ? std::atoi(v) : 0;
    }();
    sched.debug = pdebug;
    const std::size_t units = sched.full + static_cast<std::size_t>(sched.rem) * sched.nsplit;
    const std::size_t clusters = std::min<std::size_t>(units, static_cast<std::size_t>(sms / 2));
    void* ws = nullptr;
    e = split_alloc(sched, static_cast<std::size_t>(G::kLevels) * (NT / 2) * 32, stream, &ws, 2 * kPEpiWarps);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * clusters), 1);
    cfg.blockDim = dim3(kPThreads);
    cfg.dynamicSmemBytes = G::kSmem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = sched.rem > 0 ? cudaLaunchKernelEx(&cfg, ozaki_gemmp_kernel<S, NT, true>, a_sl, ea, b_sl, eb, M, N, nch, out,
                                           ld_out, col_map, fold_add, ld_add, ntn, nfast, npairs, sched)
                      : cudaLaunchKernelEx(&cfg, ozaki_gemmp_kernel<S, NT, false>, a_sl, ea, b_sl, eb, M, N, nch, out,
                                           ld_out, col_map, fold_add, ld_add, ntn, nfast, npairs, sched);
    if (ws) {
        const cudaError_t f = cudaFreeAsync(ws, stream);
        if (e == cudaSuccess) e = f;
    }
    return e;
}

template <int S, int NT, int NSUB>
cudaError_t launch_gemm2(const int8_t* a_sl, const int* ea, const int8_t* b_sl, const int* eb, std::size_t M, int N,
                         int nch, double* out, std::size_t ld_out, const int* col_map, const double* fold_add,
                         std::size_t ld_add, cudaStream_t stream) {
    using G = Geo2<S, NT>;
    cudaError_t e = smem_optin(reinterpret_cast<const void*>(ozaki_gemm2_kernel<S, NT, NSUB>), G::kSmem);
    if (e != cudaSuccess) return e;
    const std::size_t gm = (M + 2 * TM - 1) / (2 * TM) * 2; // whole CTA pairs (A rows padded to 256)
    const int ntn = (N + NT - 1) / NT;
    // tile order: the operand that is re-read per tile of the other should be
    // the one that fits in L2 — walk column tiles first when B is the smaller
    const std::size_t a_bytes = gm * TM * static_cast<std::size_t>(nch) * CB * S;
    const std::size_t b_bytes = static_cast<std::size_t>(ntn) * NT * nch * CB * S;
    static const int order = [] { // DCTP_OZAKI_ORDER: 0 = rows fastest, 1 = columns fastest, else automatic
        const char* v = std::getenv("DCTP_OZAKI_ORDER");
        return v ? std::atoi(v) : -1;
    }();
    const int nfast = order == 0 ? 0 : order == 1 ? 1 : (b_bytes < a_bytes ? 1 : 0);
    const std::size_t ntc = (static_cast<std::size_t>(ntn) + NSUB - 1) / NSUB;
    if (gm * ntc * NSUB >= (1ull << 31)) return cudaErrorInvalidValue;
    SplitSched sched;
    if (NSUB == 1) {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        plan_split(gm / 2 * ntn, static_cast<std::size_t>(sms / 2), nch, sched);
    }
    void* ws = nullptr;
    e = split_alloc(sched, static_cast<std::size_t>(G::kLevels) * NT * 32, stream, &ws);
    if (e != cudaSuccess) return e;
    const std::size_t units = sched.full + static_cast<std::size_t>(sched.rem) * sched.nsplit;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = sched.rem > 0 ? dim3(static_cast<unsigned>(2 * units), 1)
                  : (NSUB == 1 && !nfast) ? dim3(static_cast<unsigned>(gm), ntn)
                                          : dim3(static_cast<unsigned>(gm * ntc * NSUB), 1);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = G::kSmem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2 * NSUB;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    static const int debug = [] { // development knob (timing only): 1 = no loads after the first ring
        const char* v = std::getenv("DCTP_OZAKI_DEBUG");
        return v ? std::atoi(v) : 0;
    }();
    e = cudaLaunchKernelEx(&cfg, ozaki_gemm2_kernel<S, NT, NSUB>, a_sl, ea, b_sl, eb, M, N, nch, out, ld_out, col_map,
                           fold_add, ld_add, ntn, nfast, gm / 2, debug, sched);
    if (ws) {
        const cudaError_t f = cudaFreeAsync(ws, stream);
        if (e == cudaSuccess) e = f;
    }
    return e;
}

template <int S, int NT>
cudaError_t launch_gemm(const int8_t* a_sl, const int* ea, const int8_t* b_sl, const int* eb, std::size_t M, int N,
                        int nch, double* out, std::size_t ld_out, const int* col_map, const double* fold_add,
                        std::size_t ld_add, cudaStream_t stream) {
    using G = Geo<S, NT>;
    cudaError_t e = smem_optin(reinterpret_cast<const void*>(ozaki_gemm_kernel<S, NT>), G::kSmem);
    static const int debug = [] { // development knob (timing only): 1 = no loads after the first ring, 2 = no MMAs
        const char* v = std::getenv("DCTP_OZAKI_DEBUG");
        return v ? std::atoi(v) : 0;
    }();
    if (e != cudaSuccess) return e;
    const std::size_t gm = (M + TM - 1) / TM;
    const unsigned gn = static_cast<unsigned>((N + NT - 1) / NT);
    for (std::size_t m0 = 0; m0 < gm; m0 += 65535) { // grid.x limit: slices of row tiles
        const unsigned gx = static_cast<unsigned>(gm - m0 < 65535 ? gm - m0 : 65535);
        ozaki_gemm_kernel<S, NT><<<dim3(gx, gn), kThreads, G::kSmem, stream>>>(
            a_sl + m0 * nch * G::kABytes, ea + m0 * TM, b_sl, eb, M - m0 * TM, N, nch, out + m0 * TM * ld_out,
            ld_out, col_map, fold_add ? fold_add + m0 * TM * ld_add : nullptr, ld_add, debug);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

} // namespace

/// CTA-pair kernel (default; DCTP_OZAKI_PAIR=0: the single-CTA kernel);
/// DCTP_OZAKI_MCAST=1: clusters of two pairs sharing A by multicast (correct,
/// but slower: the L2 reads it saves were not the limit).
static bool pair_mode() {
    static const bool on = [] {
        const char* e = std::getenv("DCTP_OZAKI_PAIR");
        return !(e && e[0] == '0');
    }();
    return on;
}
static int pair_nsub() {
    static const int v = [] { // measured slower (C5 1.42 vs 1.36 ms, X6 0.41 vs 0.35): opt-in
        const char* e = std::getenv("DCTP_OZAKI_MCAST");
        return (e && e[0] == '1') ? 2 : 1;
    }();
    return pair_mode() ? v : 1;
}

// B rows are padded to whole clusters' column tiles
int ozaki_pad_n(int slices) { return (slices <= 5 ? 96 : 80) * pair_nsub(); }
int ozaki_tile_n(int slices) {
    const int nt = slices <= 5 ? 96 : 80;
    return pair_mode() ? nt / 2 : nt;
}
int ozaki_pad_m() { return pair_mode() ? 2 * TM : TM; }
int ozaki_group_tile(int slices) { return slices <= 5 ? 96 : 80; }

std::size_t ozaki_slice_bytes(std::size_t rows, int K, int tile_rows, int slices, int pad_rows) {
    const std::size_t pad = static_cast<std::size_t>(pad_rows > tile_rows ? pad_rows : tile_rows);
    const std::size_t tiles = (rows + pad - 1) / pad * pad / tile_rows;
    const std::size_t nch = (static_cast<std::size_t>(K) + CB - 1) / CB;
    return tiles * tile_rows * nch * CB * slices;
}

template <class T>
cudaError_t ozaki_slice(const T* in, std::size_t ld, std::size_t rows, int K, const int* a_map, int tile_rows,
                        int slices, int8_t* sl, int* expo, int* flag, cudaStream_t stream, int pad_rows) {
    if (rows == 0) return cudaSuccess;
    const std::size_t pad = static_cast<std::size_t>(pad_rows > tile_rows ? pad_rows : tile_rows);
    const std::size_t rows_pad = (rows + pad - 1) / pad * pad;
    const int nch = (K + CB - 1) / CB;
    const int vec = !a_map && reinterpret_cast<std::uintptr_t>(in) % 16 == 0 && (ld * sizeof(T)) % 16 == 0;
    if (rows_pad >= (1ull << 31)) return cudaErrorInvalidValue;
    if constexpr (sizeof(T) == 8) {
        // rows of 1025 .. 8192 samples held in registers, one CTA per row
        // (C5: 0.065 -> 0.050 ms; X8's 2048-sample rows 0.076 -> 0.048; at
        // 1024 samples half the threads would idle: 0.062 -> 0.068, so the
        // warp-per-row kernel keeps them)
        if (K > 1024 && nch * CB <= 8192 && vec && (slices == 5 || slices == 6)) {
            const int G = nch * CB <= 2048 ? 1 : (nch * CB <= 4096 ? 2 : 4);
            auto kern = slices == 5 ? (G == 1 ? ozaki_slice_reg_kernel<5, 1>
                                              : G == 2 ? ozaki_slice_reg_kernel<5, 2> : ozaki_slice_reg_kernel<5, 4>)
                                    : (G == 1 ? ozaki_slice_reg_kernel<6, 1>
                                              : G == 2 ? ozaki_slice_reg_kernel<6, 2> : ozaki_slice_reg_kernel<6, 4>);
            kern<<<static_cast<unsigned>(rows_pad), 256, 0, stream>>>(in, ld, rows, K, nch, tile_rows, sl, expo,
                                                                      flag);
            return cudaGetLastError();
        }
    }
    if (K <= 2048) // a warp per row, 8 rows per CTA
        ozaki_slice_kernel<T, 1><<<static_cast<unsigned>((rows_pad + 7) / 8), 256, 0, stream>>>(
            in, ld, rows, rows_pad, K, nch, a_map, tile_rows, slices, sl, expo, flag, vec);
    else // a CTA per row
        ozaki_slice_kernel<T, 8><<<static_cast<unsigned>(rows_pad), 256, 0, stream>>>(
            in, ld, rows, rows_pad, K, nch, a_map, tile_rows, slices, sl, expo, flag, vec);
    return cudaGetLastError();
}
template cudaError_t ozaki_slice<double>(const double*, std::size_t, std::size_t, int, const int*, int, int, int8_t*,
                                         int*, int*, cudaStream_t, int);
template cudaError_t ozaki_slice<float>(const float*, std::size_t, std::size_t, int, const int*, int, int, int8_t*,
                                        int*, int*, cudaStream_t, int);

cudaError_t ozaki_slice_fold(const double* in, std::size_t ld, std::size_t rows, int L, int tile_rows, int slices,
                             int8_t* sl, int* expo, int* flag, cudaStream_t stream, int pad_rows) {
    if (rows == 0) return cudaSuccess;
    if (L % 4 != 0 || L > 1024 || reinterpret_cast<std::uintptr_t>(in) % 16 != 0 || (ld * sizeof(double)) % 16 != 0)
        return cudaErrorInvalidValue;
    const std::size_t pad = static_cast<std::size_t>(pad_rows > tile_rows ? pad_rows : tile_rows);
    const std::size_t rows_pad = (rows + pad - 1) / pad * pad;
    const unsigned grid = static_cast<unsigned>((rows_pad + 7) / 8);
    if (slices != 5 && slices != 6) return cudaErrorInvalidValue;
    auto pick = [&](auto s5, auto s6) { return slices == 5 ? s5 : s6; };
    // register arrays sized to the row (one 128-sample step per lane group)
    auto kern = L <= 128   ? pick(ozaki_slice_fold_kernel<5, 1>, ozaki_slice_fold_kernel<6, 1>)
                : L <= 256 ? pick(ozaki_slice_fold_kernel<5, 2>, ozaki_slice_fold_kernel<6, 2>)
                : L <= 512 ? pick(ozaki_slice_fold_kernel<5, 4>, ozaki_slice_fold_kernel<6, 4>)
                           : pick(ozaki_slice_fold_kernel<5, 8>, ozaki_slice_fold_kernel<6, 8>);
    kern<<<grid, 256, 0, stream>>>(in, ld, rows, rows_pad, L, tile_rows, sl, expo, flag);
    return cudaGetLastError();
}

bool ozaki_grouped_supported() { return pair_mode() && pair_nsub() == 1; }

cudaError_t ozaki_gemm_grouped(const int8_t* a_sl, const int* ea, const int8_t* b_sl, const int* eb, std::size_t M,
                               int N, int K, int slices, double* out, std::size_t ld_out, const int* col_map,
                               int nt_split, int k_split, cudaStream_t stream) {
    if (M == 0 || N == 0) return cudaSuccess;
    if (!ozaki_grouped_supported() || k_split % CB != 0) return cudaErrorInvalidValue;
    const int nch = (K + CB - 1) / CB;
    if (slices == 5)
        return launch_gemmp<5, 96>(a_sl, ea, b_sl, eb, M, N, nch, out, ld_out, col_map, nullptr, 0, stream, nt_split,
                                   k_split / CB);
    if (slices == 6)
        return launch_gemmp<6, 80>(a_sl, ea, b_sl, eb, M, N, nch, out, ld_out, col_map, nullptr, 0, stream, nt_split,
                                   k_split / CB);
    return cudaErrorInvalidValue;
}

cudaError_t ozaki_gemm(const int8_t* a_sl, const int* ea, const int8_t* b_sl, const int* eb, std::size_t M, int N,
                       int K, int slices, double* out, std::size_t ld_out, const int* col_map, cudaStream_t stream,
                       const double* fold_add, std::size_t ld_add) {
    if (M == 0 || N == 0) return cudaSuccess;
    const int nch = (K + CB - 1) / CB;
    static const int persist = [] { // DCTP_OZAKI_PERSIST: 0 never, 1 always, else K <= 2048
        const char* e = std::getenv("DCTP_OZAKI_PERSIST");
        return e ? std::atoi(e) : -1;
    }();
    if (pair_mode() && pair_nsub() == 1 && (persist == 1 || (persist != 0 && K <= 2048))) {
        if (slices == 5)
            return launch_gemmp<5, 96>(a_sl, ea, b_sl, eb, M, N, nch, out, ld_out, col_map, fold_add, ld_add, stream);
        if (slices == 6)
            return launch_gemmp<6, 80>(a_sl, ea, b_sl, eb, M, N, nch, out, ld_out, col_map, fold_add, ld_add, stream);
        return cudaErrorInvalidValue;
    }
    if (pair_mode()) {
        const bool mc = pair_nsub() == 2;
        if (slices == 5)
            return mc ? launch_gemm2<5, 96, 2>(a_sl, ea, b_sl, eb, M, N, nch, out, ld_out, col_map, fold_add, ld_add,
                                               stream)
                      : launch_gemm2<5, 96, 1>(a_sl, ea, b_sl, eb, M, N, nch, out, ld_out, col_map, fold_add, ld_add,
                                               stream);
        if (slices == 6)
            return mc ? launch_gemm2<6, 80, 2>(a_sl, ea, b_sl, eb, M, N, nch, out, ld_out, col_map, fold_add, ld_add,
                                               stream)
                      : launch_gemm2<6, 80, 1>(a_sl, ea, b_sl, eb, M, N, nch, out, ld_out, col_map, fold_add, ld_add,
                                               stream);
        return cudaErrorInvalidValue;
    }
    if (slices == 5)
        return launch_gemm<5, 96>(a_sl, ea, b_sl, eb, M, N, nch, out, ld_out, col_map, fold_add, ld_add, stream);
    if (slices == 6)
        return launch_gemm<6, 80>(a_sl, ea, b_sl, eb, M, N, nch, out, ld_out, col_map, fold_add, ld_add, stream);
    return cudaErrorInvalidValue;
}

} // namespace dctp::dev
