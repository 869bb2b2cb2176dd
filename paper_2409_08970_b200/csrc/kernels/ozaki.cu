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

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     ptx::smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}

// ---------------------------------------------------------------- slicing

/// One CTA (8 warps) per row: pass 1 the row maximum (and the finiteness
/// check of check_signal), pass 2 the S digits.  Thread t handles 4
/// consecutive k per step (one 32-bit word of a 16-byte swizzle unit), so both
/// passes read the row with coalesced 32-byte loads (vec: 16-byte aligned
/// rows, no column map) and each slice's 64-byte chunk rows are written as
/// whole sectors; pass 2 finds the row in L1/L2.
template <class T>
__global__ void __launch_bounds__(256)
ozaki_slice_kernel(const T* __restrict__ in, std::size_t ld, std::size_t rows, int K, int nch,
                   const int* __restrict__ a_map, int tile_rows, int S, int8_t* __restrict__ sl,
                   int* __restrict__ expo, int* flag, int vec) {
    __shared__ double red[8];
    __shared__ int red_bad[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const std::size_t r = blockIdx.x;
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
    for (int k = 4 * tid; k < K; k += 1024) {
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
    const int wbad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
        red[warp] = mx;
        red_bad[warp] = wbad;
    }
    __syncthreads();
    mx = red[0];
    int anybad = red_bad[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
        mx = fmax(mx, red[w]);
        anybad |= red_bad[w];
    }
    if (anybad) {
        if (tid == 0 && flag) atomicOr(flag, 1);
        mx = 0.0;
    }
    int e = 0;
    if (mx > 0.0) frexp(mx, &e); // mx = m 2^e, m in [0.5, 1): |x| < 2^e
    if (tid == 0) expo[r] = e;
    const double scale = ldexp(127.0, -e);
    const std::size_t tile = r / tile_rows;
    const int lr = static_cast<int>(r % tile_rows);
    const std::size_t slice_bytes = static_cast<std::size_t>(tile_rows) * CB;
#pragma unroll 2
    for (int k = 4 * tid; k < nch * CB; k += 1024) {
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
                const double d = rint(v[u]);
                v[u] = (v[u] - d) * 254.0;
                w |= (static_cast<uint32_t>(static_cast<int>(d)) & 0xFFu) << (8 * u);
            }
            *reinterpret_cast<uint32_t*>(dst + s * slice_bytes) = w;
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

template <int S, int NT>
__global__ void __launch_bounds__(kThreads, 1)
ozaki_gemm_kernel(const int8_t* __restrict__ a_sl, const int* __restrict__ ea, const int8_t* __restrict__ b_sl,
                  const int* __restrict__ eb, std::size_t M, int N, int nch, double* __restrict__ out,
                  std::size_t ld_out, const int* __restrict__ col_map, const double* __restrict__ fold_add,
                  std::size_t ld_add) {
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

    if (warp == 0) {
        if (lane == 0) { // producer: one A and one B bulk copy per chunk
            for (int ch = 0; ch < nch; ++ch) {
                const int st = ch % G::kStages;
                if (ch >= G::kStages) ptx::mbar_wait(empty + st, static_cast<uint32_t>(((ch / G::kStages) - 1) & 1));
                ptx::mbar_expect_tx(full + st, G::kStageBytes);
                unsigned char* dst = base + st * G::kStageBytes;
                ptx::bulk_load(dst, a_tile + static_cast<std::size_t>(ch) * G::kABytes, G::kABytes, full + st);
                ptx::bulk_load(dst + G::kABytes, b_tile + static_cast<std::size_t>(ch) * G::kBBytes, G::kBBytes,
                               full + st);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) { // MMA issuer
            for (int ch = 0; ch < nch; ++ch) {
                const int st = ch % G::kStages;
                ptx::mbar_wait(full + st, static_cast<uint32_t>((ch / G::kStages) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                const uint32_t sa = sbase + st * G::kStageBytes, sb = sa + G::kABytes;
#pragma unroll
                for (int kk = 0; kk < CB / 32; ++kk) {
                    const uint32_t o = 32u * kk;
#pragma unroll
                    for (int L = 0; L < G::kLevels; ++L) {
                        const uint32_t td = tmem + static_cast<uint32_t>(L * NT);
#pragma unroll
                        for (int i = 0; i <= L; ++i) {
                            const int j = L - i;
                            const uint32_t acc = (ch > 0 || kk > 0 || i > 0) ? 1u : 0u;
                            mma_i8<NT>(td, smem_desc(sa + i * TM * CB + o), smem_desc(sb + j * NT * CB + o), acc);
                        }
                    }
                }
                mma_commit(empty + st);
            }
            mma_commit(done);
        }
        __syncwarp();
    }

    // epilogue: warp w reads TMEM lanes 32 w .. 32 w + 31 (tile rows)
    ptx::mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const std::size_t row = mt * TM + 32 * warp + lane;
    const bool live = row < M;
    const double rs = live ? ldexp(1.0 / (127.0 * 127.0), ea[row]) : 0.0;
    constexpr double kInv = 1.0 / 254.0;
#pragma unroll 1
    for (int c0 = 0; c0 < NT; c0 += 32) {
        double acc[32];
        uint32_t v[32];
#pragma unroll 1
        for (int L = G::kLevels - 1; L >= 0; --L) {
            tmem_ld32(tmem + (static_cast<uint32_t>(32 * warp) << 16) + static_cast<uint32_t>(L * NT + c0), v);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            if (L == G::kLevels - 1) {
#pragma unroll
                for (int u = 0; u < 32; ++u) acc[u] = static_cast<double>(static_cast<int>(v[u]));
            } else {
#pragma unroll
                for (int u = 0; u < 32; ++u) acc[u] = fma(acc[u], kInv, static_cast<double>(static_cast<int>(v[u])));
            }
        }
        if (live) {
            const int cbase = nt * NT + c0;
            const int lim = min(N, nt * NT + NT); // columns of this tile
            double* orow = out + row * ld_out;
            if (fold_add) { // unfold: x_c = w_c + v_c, x_{2N-1-c} = w_c - v_c
                const double* add = fold_add + row * ld_add;
#pragma unroll 4
                for (int u = 0; u < 32; ++u)
                    if (cbase + u < lim) {
                        const double v = acc[u] * ldexp(rs, __ldg(eb + cbase + u)), w = add[cbase + u];
                        orow[cbase + u] = w + v;
                        orow[2 * N - 1 - (cbase + u)] = w - v;
                    }
            } else if (col_map) {
#pragma unroll
                for (int u = 0; u < 32; ++u)
                    if (cbase + u < lim) orow[__ldg(col_map + cbase + u)] = acc[u] * ldexp(rs, __ldg(eb + cbase + u));
            } else if (cbase + 32 <= lim && (ld_out & 1) == 0) {
#pragma unroll
                for (int u = 0; u < 32; u += 2)
                    *reinterpret_cast<double2*>(orow + cbase + u) =
                        make_double2(acc[u] * ldexp(rs, __ldg(eb + cbase + u)),
                                     acc[u + 1] * ldexp(rs, __ldg(eb + cbase + u + 1)));
            } else {
#pragma unroll
                for (int u = 0; u < 32; ++u)
                    if (cbase + u < lim) orow[cbase + u] = acc[u] * ldexp(rs, __ldg(eb + cbase + u));
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
}

template <int S, int NT>
cudaError_t launch_gemm(const int8_t* a_sl, const int* ea, const int8_t* b_sl, const int* eb, std::size_t M, int N,
                        int nch, double* out, std::size_t ld_out, const int* col_map, const double* fold_add,
                        std::size_t ld_add, cudaStream_t stream) {
    using G = Geo<S, NT>;
    cudaError_t e = smem_optin(reinterpret_cast<const void*>(ozaki_gemm_kernel<S, NT>), G::kSmem);
    if (e != cudaSuccess) return e;
    const std::size_t gm = (M + TM - 1) / TM;
    const unsigned gn = static_cast<unsigned>((N + NT - 1) / NT);
    for (std::size_t m0 = 0; m0 < gm; m0 += 65535) { // grid.x limit: slices of row tiles
        const unsigned gx = static_cast<unsigned>(gm - m0 < 65535 ? gm - m0 : 65535);
        ozaki_gemm_kernel<S, NT><<<dim3(gx, gn), kThreads, G::kSmem, stream>>>(
            a_sl + m0 * nch * G::kABytes, ea + m0 * TM, b_sl, eb, M - m0 * TM, N, nch, out + m0 * TM * ld_out,
            ld_out, col_map, fold_add ? fold_add + m0 * TM * ld_add : nullptr, ld_add);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

} // namespace

int ozaki_tile_n(int slices) { return slices <= 5 ? 96 : 80; }

std::size_t ozaki_slice_bytes(std::size_t rows, int K, int tile_rows, int slices) {
    const std::size_t tiles = (rows + tile_rows - 1) / tile_rows;
    const std::size_t nch = (static_cast<std::size_t>(K) + CB - 1) / CB;
    return tiles * tile_rows * nch * CB * slices;
}

template <class T>
cudaError_t ozaki_slice(const T* in, std::size_t ld, std::size_t rows, int K, const int* a_map, int tile_rows,
                        int slices, int8_t* sl, int* expo, int* flag, cudaStream_t stream) {
    if (rows == 0) return cudaSuccess;
    const std::size_t rows_pad = (rows + tile_rows - 1) / tile_rows * tile_rows;
    const int nch = (K + CB - 1) / CB;
    const int vec = !a_map && reinterpret_cast<std::uintptr_t>(in) % 16 == 0 && (ld * sizeof(T)) % 16 == 0;
    if (rows_pad >= (1ull << 31)) return cudaErrorInvalidValue; // one CTA per (padded) row
    ozaki_slice_kernel<T><<<static_cast<unsigned>(rows_pad), 256, 0, stream>>>(in, ld, rows, K, nch, a_map, tile_rows,
                                                                               slices, sl, expo, flag, vec);
    return cudaGetLastError();
}
template cudaError_t ozaki_slice<double>(const double*, std::size_t, std::size_t, int, const int*, int, int, int8_t*,
                                         int*, int*, cudaStream_t);
template cudaError_t ozaki_slice<float>(const float*, std::size_t, std::size_t, int, const int*, int, int, int8_t*,
                                        int*, int*, cudaStream_t);

cudaError_t ozaki_gemm(const int8_t* a_sl, const int* ea, const int8_t* b_sl, const int* eb, std::size_t M, int N,
                       int K, int slices, double* out, std::size_t ld_out, const int* col_map, cudaStream_t stream,
                       const double* fold_add, std::size_t ld_add) {
    if (M == 0 || N == 0) return cudaSuccess;
    const int nch = (K + CB - 1) / CB;
    if (slices == 5)
        return launch_gemm<5, 96>(a_sl, ea, b_sl, eb, M, N, nch, out, ld_out, col_map, fold_add, ld_add, stream);
    if (slices == 6)
        return launch_gemm<6, 80>(a_sl, ea, b_sl, eb, M, N, nch, out, ld_out, col_map, fold_add, ld_add, stream);
    return cudaErrorInvalidValue;
}

} // namespace dctp::dev
