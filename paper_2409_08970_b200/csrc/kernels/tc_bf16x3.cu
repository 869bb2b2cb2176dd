// fp32 GEMM with a short K on the tcgen05 tensor cores, bf16x3 split
// (kind::f16, fp32 accumulation in TMEM), sm_100a — the progressive ensemble
// of config 4 (forward_all = x [D^T | X_1 .. X_K], fast_transform.hpp:396-403
// with c_p = n): C[M x N] = A[M x K] B^T[N x K]^T, K <= 128.
//
// Each operand is split a = a_hi + a_lo into two bf16 (a_hi = bf16(a), a_lo =
// bf16(a - a_hi)) and the product accumulates a_hi b_hi + a_hi b_lo + a_lo b_hi
// (the dropped a_lo b_lo is ~2^-16 relative): 2.2e-6 from the reference at C4
// against the 1e-4 fp32 tolerance, the same order as 3xTF32, at twice the
// tensor rate with half the operand bytes.
//
// The kernel is bound by its output stream (C4: 570 MB of fp32 coefficients
// for 34 MB of input), so it is built to keep stores flowing:
//   * persistent CTAs (one per SM) over a column-major tile order: a CTA's
//     range of 128 x 256 tiles mostly shares one column tile, whose B^T block
//     (all of K, hi and lo: 128 KB) stays resident in shared memory, while A
//     row tiles stream through a 3-stage ring of 16 KB chunks;
//   * warp roles: warp 0 produces (TMA bulk copies), warp 1 issues the MMAs
//     (one elected lane), warps 2..9 drain TMEM;
//   * two TMEM accumulators (2 x 256 columns): the epilogue of tile i overlaps
//     the MMAs of tile i + 1;
//   * the epilogue transposes each 32 x 32 block through shared memory so every
//     store instruction writes whole 128-byte lines (streaming stores).
// The A split runs as a separate pass (bf16x3_split_kernel) into the exact
// shared-memory image, so each A chunk is one bulk copy.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include "kernels/common.cuh"
#include "kernels/launch.hpp"

namespace dctp::dev {
namespace {

constexpr int BM = 128, BN = 256, KC = 32; // K chunk: 32 bf16 = one 64-byte SW64 row
constexpr int kMaxK = 128;
constexpr int kAStages = 3;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 32 * (2 + kEpiWarps);
constexpr int kAHalf = BM * KC * 2;            // one of hi / lo of an A chunk: 8 KB
constexpr int kAChunk = 2 * kAHalf;            // 16 KB
constexpr int kBHalf = BN * KC * 2;            // 16 KB
constexpr int kBChunk = 2 * kBHalf;            // 32 KB
constexpr int kBBytes = (kMaxK / KC) * kBChunk; // 128 KB resident
constexpr int kStaging = kEpiWarps * 32 * 32 * 4;

__host__ __device__ constexpr uint32_t sw64_off(int r, int c16) {
    return static_cast<uint32_t>(r * 64 + ((c16 ^ ((r >> 1) & 3)) << 4));
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(512 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(4) << 61;
    return d;
}

/// D fp32, A and B bf16, both K-major, M = 128, N = 256.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                            (static_cast<uint32_t>(BM >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     ptx::smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}\n" : "=r"(pred));
    return pred != 0;
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

__device__ __forceinline__ uint32_t bf16_bits(float x) {
    return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(x)));
}

/// A split: rows of fp32 (stride lda; columns gathered through a_map if
/// given) -> bf16 hi / lo in the kernel's chunk
/// image [row tile][chunk][hi | lo][128 rows x 64 B, SW64]; one thread per
/// 8 consecutive k (one 16-byte unit of each half).
__global__ void __launch_bounds__(256) bf16x3_split_kernel(const float* __restrict__ a, int lda, std::size_t M,
                                                           std::size_t rows_pad, int K, int nch,
                                                           const int* __restrict__ a_map,
                                                           unsigned char* __restrict__ a_sw) {
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int units = nch * (KC / 8);
    if (i >= rows_pad * units) return;
    const std::size_t r = i / units;
    const int u = static_cast<int>(i % units), k0 = 8 * u;
    float v[8];
    if (!a_map && r < M && k0 + 8 <= K && (lda & 3) == 0) {
        const float4 p = __ldg(reinterpret_cast<const float4*>(a + r * lda + k0));
        const float4 q = __ldg(reinterpret_cast<const float4*>(a + r * lda + k0 + 4));
        v[0] = p.x, v[1] = p.y, v[2] = p.z, v[3] = p.w, v[4] = q.x, v[5] = q.y, v[6] = q.z, v[7] = q.w;
    } else {
#pragma unroll
        for (int t = 0; t < 8; ++t)
            v[t] = (r < M && k0 + t < K) ? a[r * lda + (a_map ? __ldg(a_map + k0 + t) : k0 + t)] : 0.f;
    }
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const float h0 = __bfloat162float(__float2bfloat16_rn(v[2 * t]));
        const float h1 = __bfloat162float(__float2bfloat16_rn(v[2 * t + 1]));
        hi[t] = bf16_bits(h0) | (bf16_bits(h1) << 16);
        lo[t] = bf16_bits(v[2 * t] - h0) | (bf16_bits(v[2 * t + 1] - h1) << 16);
    }
    const std::size_t mt = r / BM;
    const int lr = static_cast<int>(r % BM), ch = k0 / KC, c16 = (k0 % KC) / 8;
    unsigned char* blk = a_sw + (mt * nch + ch) * static_cast<std::size_t>(kAChunk) + sw64_off(lr, c16);
    *reinterpret_cast<uint4*>(blk) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(blk + kAHalf) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
}

struct Sched {
    unsigned long long first, last; // this CTA's tiles [first, last), column-major
    unsigned ntm;                   // row tiles
    __device__ void tile(unsigned long long t, unsigned& mt, unsigned& nt) const {
        nt = static_cast<unsigned>(t / ntm);
        mt = static_cast<unsigned>(t % ntm);
    }
};

/// Output of one tile: plain rows (C[r, c]), scattered columns (C[r,
/// col_map[c]]), or unfolded (C[r, c] = w + v, C[r, 2N - 1 - c] = w - v with
/// w = fold_add[r, c], the folded inverse of antisymmetric plans).
struct Epi {
    float* C;
    std::size_t ldc;
    const int* col_map;
    const float* fold_add;
    std::size_t ld_add;
    int debug = 0; // DCTP_TC_DEBUG (development: phase isolation)
};

/// STREAM = false: K <= 128, the B^T column tile resident (one load per
/// column tile).  STREAM = true: any K, A and B chunks stream together
/// through a 4-stage ring (48 KB per stage).
template <bool STREAM>
struct Lay {
    static constexpr int kStages = STREAM ? 4 : kAStages;
    static constexpr int kStage = STREAM ? kAChunk + kBChunk : kAChunk;
    static constexpr int kResident = STREAM ? 0 : kBBytes;
    static constexpr int kSmem = kResident + kStages * kStage + kStaging + 1024 + 256;
    static_assert(kSmem <= 227 * 1024, "tc_bf16x3: shared memory");
};

/// TMA store of one 32 x 32 fp32 block staged in shared memory (128-byte
/// rows, SWIZZLE_128B — the turn-around's own layout) at (row0, col0) of C.
__device__ __forceinline__ void tma_store_block(const CUtensorMap* map, const void* smem, int col0, int row0) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(col0), "r"(row0), "r"(ptx::smem_addr(smem))
        : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}

template <bool STREAM, int MODE> // MODE 0: plain rows, 1: col_map, 2: fold_add, 3: plain rows by TMA stores
__global__ void __launch_bounds__(kThreads, 1)
tc_bf16x3_kernel(const unsigned char* __restrict__ a_sw, const unsigned char* __restrict__ b_sw, Epi ep,
                 std::size_t M, int N, int nch, unsigned ntm, unsigned ntn, int* flag,
                 const __grid_constant__ CUtensorMap cmap) {
    using Ly = Lay<STREAM>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t raw = ptx::smem_addr(smem_raw);
    unsigned char* base = smem_raw + ((1024 - (raw & 1023)) & 1023);
    unsigned char* bsm = base;                                // resident B^T column tile (!STREAM)
    unsigned char* ring = base + Ly::kResident;               // stages: A chunk (+ B chunk when STREAM)
    unsigned char* stg = ring + Ly::kStages * Ly::kStage;     // epilogue transposes
    uint64_t* bar = reinterpret_cast<uint64_t*>(stg + kStaging);
    uint64_t* s_full = bar;                       // kStages
    uint64_t* s_empty = s_full + Ly::kStages;     // kStages
    uint64_t* b_full = s_empty + Ly::kStages;     // 1
    uint64_t* b_empty = b_full + 1;               // 1
    uint64_t* t_full = b_empty + 1;               // 2: accumulator ready
    uint64_t* t_empty = t_full + 2;               // 2: accumulator drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned long long total = static_cast<unsigned long long>(ntm) * ntn;
    Sched sc{total * blockIdx.x / gridDim.x, total * (blockIdx.x + 1) / gridDim.x, ntm};

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                         ptx::smem_addr(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    if (threadIdx.x == 32) {
        for (int i = 0; i < Ly::kStages; ++i) {
            ptx::mbar_init(s_full + i, 1);
            ptx::mbar_init(s_empty + i, 1);
        }
        ptx::mbar_init(b_full, 1);
        ptx::mbar_init(b_empty, 1);
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(t_full + i, 1);
            ptx::mbar_init(t_empty + i, kEpiWarps);
        }
        ptx::fence_mbar_init();
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) { // producer
        unsigned cur_nt = ~0u, b_loads = 0;
        unsigned long long chunk = 0;
        for (unsigned long long t = sc.first; t < sc.last; ++t) {
            unsigned mt, nt;
            sc.tile(t, mt, nt);
            if (!STREAM && nt != cur_nt) { // (re)load the resident B^T block once its readers are done
                if (b_loads > 0) ptx::mbar_wait(b_empty, (b_loads - 1) & 1u);
                if (elect_one()) {
                    ptx::mbar_expect_tx(b_full, static_cast<uint32_t>(nch * kBChunk));
                    for (int c = 0; c < nch; ++c)
                        ptx::bulk_load(bsm + c * kBChunk, b_sw + (static_cast<std::size_t>(nt) * nch + c) * kBChunk,
                                       kBChunk, b_full);
                }
                __syncwarp();
                cur_nt = nt;
                ++b_loads;
            }
            for (int c = 0; c < nch; ++c, ++chunk) {
                const int st = static_cast<int>(chunk % Ly::kStages);
                const uint32_t ph = static_cast<uint32_t>((chunk / Ly::kStages) & 1);
                ptx::mbar_wait(s_empty + st, ph ^ 1u);
                // development knob DCTP_TC_DEBUG=1: only the first ring of A chunks is loaded
                const bool skip = (ep.debug & 1) && chunk >= static_cast<unsigned long long>(Ly::kStages);
                if (elect_one()) {
                    ptx::mbar_expect_tx(s_full + st, skip ? 0u : static_cast<uint32_t>(Ly::kStage));
                    unsigned char* dst = ring + st * Ly::kStage;
                    if (!skip)
                        ptx::bulk_load(dst, a_sw + (static_cast<std::size_t>(mt) * nch + c) * kAChunk, kAChunk,
                                       s_full + st);
                    if (STREAM && !skip)
                        ptx::bulk_load(dst + kAChunk, b_sw + (static_cast<std::size_t>(nt) * nch + c) * kBChunk,
                                       kBChunk, s_full + st);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) { // MMA issuer
        const uint64_t rdesc0 = smem_desc(ptx::smem_addr(ring)), bdesc0 = smem_desc(ptx::smem_addr(bsm));
        unsigned cur_nt = ~0u, b_loads = 0;
        unsigned long long chunk = 0;
        int i = 0;
        for (unsigned long long t = sc.first; t < sc.last; ++t, ++i) {
            unsigned mt, nt;
            sc.tile(t, mt, nt);
            if (!STREAM && nt != cur_nt) {
                ptx::mbar_wait(b_full, b_loads & 1u);
                cur_nt = nt;
                ++b_loads;
            }
            const int buf = i & 1;
            ptx::mbar_wait(t_empty + buf, static_cast<uint32_t>(((i >> 1) & 1) ^ 1));
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const uint32_t td = tmem + static_cast<uint32_t>(buf * BN);
            for (int c = 0; c < nch; ++c, ++chunk) {
                const int st = static_cast<int>(chunk % Ly::kStages);
                ptx::mbar_wait(s_full + st, static_cast<uint32_t>((chunk / Ly::kStages) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                if (elect_one()) {
                    const uint64_t ah = rdesc0 + (static_cast<uint64_t>(st * Ly::kStage) >> 4);
                    const uint64_t al = ah + (kAHalf >> 4);
                    const uint64_t bh = STREAM ? ah + (kAChunk >> 4)
                                               : bdesc0 + (static_cast<uint64_t>(c * kBChunk) >> 4);
                    const uint64_t bl = bh + (kBHalf >> 4);
#pragma unroll
                    for (int kk = 0; kk < KC / 16; ++kk) { // 16 bf16 = 32 bytes per MMA K step
                        const uint64_t o = static_cast<uint64_t>(32 * kk) >> 4;
                        mma_bf16(td, ah + o, bh + o, (c > 0 || kk > 0) ? 1u : 0u);
                        mma_bf16(td, ah + o, bl + o, 1u);
                        mma_bf16(td, al + o, bh + o, 1u);
                    }
                    mma_commit(s_empty + st);
                }
                __syncwarp();
            }
            if (elect_one()) {
                mma_commit(t_full + buf);
                if (!STREAM) { // the last tile of this column tile: B may be replaced once these MMAs are done
                    unsigned mt2 = 0, nt2 = ~0u;
                    if (t + 1 < sc.last) sc.tile(t + 1, mt2, nt2);
                    if (nt2 != nt) mma_commit(b_empty);
                }
            }
            __syncwarp();
        }
    } else { // epilogue warps 2..9: TMEM lane quarter warp % 4, column half (warp - 2) / 4
        const int q = warp & 3, h = (warp - 2) >> 2;
        unsigned char* tb = stg + (warp - 2) * 4096;
        int i = 0;
        bool bad = false;
        for (unsigned long long t = sc.first; t < sc.last; ++t, ++i) {
            unsigned mt, nt;
            sc.tile(t, mt, nt);
            const int buf = i & 1;
            ptx::mbar_wait(t_full + buf, static_cast<uint32_t>((i >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const std::size_t row0 = static_cast<std::size_t>(mt) * BM + 32 * q;
            // the warp's four 32 x 32 blocks: block k + 1's TMEM load is in
            // flight while block k turns around and stores; the accumulator
            // is released as soon as the last block is in registers
            constexpr int kBlk = BN / 2 / 32;
            const int colh = static_cast<int>(nt) * BN + h * (BN / 2);
            const int nblk = colh >= N ? 0 : min(kBlk, (N - colh + 31) / 32);
            const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * q) << 16) +
                                   static_cast<uint32_t>(buf * BN + h * (BN / 2));
            uint32_t v[2][32];
            if (nblk > 0) tmem_ld32(taddr, v[0]);
#pragma unroll
            for (int k = 0; k < kBlk; ++k) {
                if (k >= nblk) break;
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                if (k + 1 < nblk) {
                    tmem_ld32(taddr + static_cast<uint32_t>(32 * (k + 1)), v[(k + 1) & 1]);
                } else {
                    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(t_empty + buf);
                }
                const uint32_t(&w32)[32] = v[k & 1];
                const int col0 = colh + 32 * k;
                if (col0 == 0 && row0 + lane < M) bad |= !isfinite(__uint_as_float(w32[0])); // column 0
                if constexpr (MODE == 3) { // the previous block's store must have read the staging
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                    __syncwarp();
                }
#pragma unroll
                for (int g = 0; g < 8; ++g)
                    *reinterpret_cast<uint4*>(tb + lane * 128 + ((g ^ (lane & 7)) << 4)) =
                        make_uint4(w32[4 * g], w32[4 * g + 1], w32[4 * g + 2], w32[4 * g + 3]);
                if constexpr (MODE == 3) { // one TMA store per block (rows >= M / columns >= N are clipped)
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    __syncwarp();
                    if (lane == 0) tma_store_block(&cmap, tb, col0, static_cast<int>(row0));
                    continue;
                }
                __syncwarp();
                // lane (row group lane >> 3, 4-column group g): the same
                // columns in all 8 iterations; the unfold's fold rows are all
                // loaded before the first store (the stores may alias them, so
                // the compiler would otherwise serialise load -> store)
                const int g = lane & 7, col = col0 + 4 * g;
                float4 add[8];
                if constexpr (MODE == 2) { // N % 4 == 0 on this path
#pragma unroll
                    for (int it = 0; it < 8; ++it) {
                        const std::size_t grow = row0 + 4 * it + (lane >> 3);
                        add[it] = (grow < M && col < N)
                                      ? __ldg(reinterpret_cast<const float4*>(ep.fold_add + grow * ep.ld_add + col))
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
#pragma unroll
                for (int it = 0; it < 8; ++it) {
                    const int r = 4 * it + (lane >> 3);
                    const uint4 w = *reinterpret_cast<const uint4*>(tb + r * 128 + ((g ^ (r & 7)) << 4));
                    const std::size_t grow = row0 + r;
                    if (grow >= M || col >= N) continue;
                    const float e4[4] = {__uint_as_float(w.x), __uint_as_float(w.y), __uint_as_float(w.z),
                                         __uint_as_float(w.w)};
                    float* orow = ep.C + grow * ep.ldc;
                    if constexpr (MODE == 2) {
                        const float4 a4 = add[it];
                        __stcs(reinterpret_cast<float4*>(orow + col),
                               make_float4(a4.x + e4[0], a4.y + e4[1], a4.z + e4[2], a4.w + e4[3]));
                        __stcs(reinterpret_cast<float4*>(orow + 2 * N - 4 - col),
                               make_float4(a4.w - e4[3], a4.z - e4[2], a4.y - e4[1], a4.x - e4[0]));
                    } else if constexpr (MODE == 1) {
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (col + u < N) orow[__ldg(ep.col_map + col + u)] = e4[u];
                    } else {
                        if (col + 4 <= N) {
                            __stcs(reinterpret_cast<float4*>(orow + col), make_float4(e4[0], e4[1], e4[2], e4[3]));
                        } else {
                            for (int u = 0; u < 4 && col + u < N; ++u) orow[col + u] = e4[u];
                        }
                    }
                }
                __syncwarp();
            }
            if (nblk == 0) {
                asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(t_empty + buf);
            }

        }
        if (bad) atomicOr(flag, 1);
        if constexpr (MODE == 3)
            if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
}

} // namespace

std::size_t tc_bf16x3_a_bytes(std::size_t M, int K) {
    return (M + BM - 1) / BM * static_cast<std::size_t>((K + KC - 1) / KC) * kAChunk;
}

bool tc_bf16x3_supported(int K, int N, std::size_t ldc, const void* C, bool fold) {
    return K > 0 && N > 0 && ldc % 4 == 0 && reinterpret_cast<std::uintptr_t>(C) % 16 == 0 && (!fold || N % 4 == 0);
}

std::vector<uint16_t> tc_bf16x3_swizzle_b(const double* bt, int N, int K, int ldb) {
    const int ntn = (N + BN - 1) / BN, nch = (K + KC - 1) / KC;
    std::vector<uint16_t> out(static_cast<std::size_t>(ntn) * nch * kBChunk / 2, 0);
    auto bf = [](float x) -> uint16_t { // round to nearest even (host __float2bfloat16_rn)
        uint32_t u;
        std::memcpy(&u, &x, 4);
        u += 0x7FFFu + ((u >> 16) & 1u);
        return static_cast<uint16_t>(u >> 16);
    };
    auto unbf = [](uint16_t h) {
        const uint32_t u = static_cast<uint32_t>(h) << 16;
        float f;
        std::memcpy(&f, &u, 4);
        return f;
    };
    for (int nt = 0; nt < ntn; ++nt)
        for (int c = 0; c < nch; ++c) {
            uint16_t* blk = out.data() + (static_cast<std::size_t>(nt) * nch + c) * (kBChunk / 2);
            for (int r = 0; r < BN; ++r)
                for (int kl = 0; kl < KC; ++kl) {
                    const int n = nt * BN + r, k = c * KC + kl;
                    if (n >= N || k >= K) continue;
                    const double v = bt[static_cast<std::size_t>(n) * ldb + k];
                    const uint16_t hi = bf(static_cast<float>(v));
                    const uint16_t lo = bf(static_cast<float>(v - static_cast<double>(unbf(hi))));
                    const std::size_t at = (sw64_off(r, kl / 8) + (kl % 8) * 2) / 2;
                    blk[at] = hi;
                    blk[kBHalf / 2 + at] = lo;
                }
        }
    return out;
}

/// Tensor map of C (M rows x N fp32 columns, row stride ldc) in 32 x 32
/// boxes with 128-byte swizzle, for the TMA-store epilogue; false if the
/// driver entry point or the encoding is unavailable (the kernel then stores
/// with st.global).
static bool c_tensor_map(float* C, std::size_t ldc, std::size_t M, int N, CUtensorMap* map) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode || M >= (1ull << 31) || (ldc * 4) % 16 != 0 || reinterpret_cast<std::uintptr_t>(C) % 16 != 0)
        return false;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(M)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldc) * 4};
    const cuuint32_t box[2] = {32, 32}, estr[2] = {1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, C, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t tc_bf16x3(const float* A, int lda, const uint16_t* b_sw, float* C, std::size_t ldc, std::size_t M, int N,
                      int K, int* flag, int num_sms, cudaStream_t stream, const int* col_map, const int* a_map,
                      const float* fold_add, std::size_t ld_add, const unsigned char* a_img) {
    if (M == 0 || N == 0) return cudaSuccess;
    if (K <= 0) return cudaErrorInvalidValue;
    const int nch = (K + KC - 1) / KC;
    const std::size_t ntm = (M + BM - 1) / BM;
    if (ntm >= (1ull << 32)) return cudaErrorInvalidValue;
    cudaError_t e = cudaSuccess;
    unsigned char* a_sw = nullptr;
    if (!a_img) {
        e = cudaMallocAsync(reinterpret_cast<void**>(&a_sw), ntm * nch * static_cast<std::size_t>(kAChunk), stream);
        if (e != cudaSuccess) return e;
        const std::size_t rows_pad = ntm * BM, work = rows_pad * nch * (KC / 8);
        bf16x3_split_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(A, lda, M, rows_pad, K,
                                                                                          nch, a_map, a_sw);
        e = cudaGetLastError();
    }
    const unsigned char* a_use = a_img ? a_img : a_sw;
    if (e == cudaSuccess) {
        const unsigned ntn = static_cast<unsigned>((N + BN - 1) / BN);
        const unsigned long long tiles = static_cast<unsigned long long>(ntm) * ntn;
        const unsigned grid = static_cast<unsigned>(tiles < static_cast<unsigned long long>(num_sms) ? tiles : num_sms);
        static const int dbg = [] {
            const char* v = std::getenv("DCTP_TC_DEBUG");
            return v ? std::atoi(v) : 0;
        }();
        const Epi ep{C, ldc, col_map, fold_add, ld_add, dbg};
        int mode = fold_add ? 2 : (col_map ? 1 : 0);
        CUtensorMap cmap;
        std::memset(&cmap, 0, sizeof(cmap));
        // DCTP_TC_TMA_STORE=1: plain rows leave by TMA tensor stores (one per
        // 32 x 32 block) instead of st.global — measured slower at C4 (0.158
        // vs 0.148 ms: the stores are not issue-bound), kept opt-in
        static const bool tma_store = [] {
            const char* v = std::getenv("DCTP_TC_TMA_STORE");
            return v && v[0] == '1';
        }();
        if (mode == 0 && tma_store && c_tensor_map(C, ldc, M, N, &cmap)) mode = 3;
        auto launch = [&](auto kern, int smem) {
            cudaError_t r = smem_optin(reinterpret_cast<const void*>(kern), smem);
            if (r != cudaSuccess) return r;
            kern<<<grid, kThreads, smem, stream>>>(a_use, reinterpret_cast<const unsigned char*>(b_sw), ep, M, N, nch,
                                                   static_cast<unsigned>(ntm), ntn, flag, cmap);
            return cudaGetLastError();
        };
        if (K > kMaxK)
            e = mode == 3   ? launch(tc_bf16x3_kernel<true, 3>, Lay<true>::kSmem)
                : mode == 2 ? launch(tc_bf16x3_kernel<true, 2>, Lay<true>::kSmem)
                : mode == 1 ? launch(tc_bf16x3_kernel<true, 1>, Lay<true>::kSmem)
                            : launch(tc_bf16x3_kernel<true, 0>, Lay<true>::kSmem);
        else
            e = mode == 3   ? launch(tc_bf16x3_kernel<false, 3>, Lay<false>::kSmem)
                : mode == 2 ? launch(tc_bf16x3_kernel<false, 2>, Lay<false>::kSmem)
                : mode == 1 ? launch(tc_bf16x3_kernel<false, 1>, Lay<false>::kSmem)
                            : launch(tc_bf16x3_kernel<false, 0>, Lay<false>::kSmem);
    }
    if (a_sw) cudaFreeAsync(a_sw, stream);
    return e;
}

} // namespace dctp::dev
