// fp32 GEMM on the 5th-generation tensor cores (tcgen05, kind::tf32) with the
// 3xTF32 split, sm_100a:  C[M x N] = A[M x K] * B[K x N], A row-major fp32,
// B given transposed and pre-split (bt_hi + bt_lo, N x K, K contiguous).
//
// Used for the fp32 progressive ensembles (C4: forward_all = x [D^T | X_1 ..
// X_K], fast_transform.hpp:396-403 with c_p = n), where the FFMA SGEMM is
// FMA-bound at ~67% of the CUDA-core peak.  Each operand is split into a
// TF32 head and an fp32 tail, a = a_hi + a_lo, and the product accumulates
// a_hi b_hi + a_hi b_lo + a_lo b_hi in fp32 in TMEM (the a_lo b_lo term is
// below fp32 rounding): ~fp32 accuracy, against the 1e-4 fp32 tolerance.
//
// CTA tile 128 x 256, K in 16-wide chunks (one 64-byte swizzle atom of fp32)
// through a two-stage ring: A chunks are split in registers and stored hi /
// lo into SWIZZLE_64B K-major shared memory, B chunks (hi, lo) arrive by
// cp.async into the same layout, and chunk k + 1 loads while the tensor core
// runs chunk k.  One thread issues the 2 x 3 tcgen05.mma of a chunk and
// commits them to the stage's mbarrier; the accumulator (128 lanes x 256
// fp32 columns) lives in TMEM and leaves through tcgen05.ld, one row per
// thread, as full 32-byte sectors.  96 KB of shared memory: two CTAs per SM,
// so one CTA's epilogue overlaps the other's loads and MMAs.
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "kernels/common.cuh"
#include "kernels/launch.hpp"

namespace dctp::dev {
namespace {

constexpr int BM = 128, BN = 256, BK = 16, kStages = 2;
constexpr int kThreads = 128;
constexpr uint32_t kTmemCols = 256;
constexpr int kABytes = BM * BK * 4, kBBytes = BN * BK * 4;          // 8 KB, 16 KB
constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;                 // A hi, A lo, B hi, B lo: 48 KB
constexpr int kSmem = kStages * kStageBytes + 1024 + 64;               // + alignment slack, barriers, tmem slot

/// Byte offset of (row r, 16-byte chunk c) in a K-major SWIZZLE_64B tile whose
/// rows are one 64-byte atom wide (16 fp32; 8-row groups of 512 bytes):
/// Swizzle<2,4,3>, the chunk index XORed with address bits 7-8.
__device__ __forceinline__ uint32_t sw64(int r, int c) {
    return static_cast<uint32_t>(r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
}

/// Shared-memory matrix descriptor (tcgen05): K-major, SWIZZLE_64B, SBO = 512
/// bytes between 8-row groups, LBO unused (1), version 1.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
    d |= static_cast<uint64_t>(1) << 16;             // leading byte offset (ignored for swizzled K-major)
    d |= static_cast<uint64_t>(512 >> 4) << 32;      // stride byte offset
    d |= static_cast<uint64_t>(1) << 46;             // descriptor version (sm_100)
    d |= static_cast<uint64_t>(4) << 61;             // SWIZZLE_64B
    return d;
}

/// Instruction descriptor: D fp32, A and B tf32, both K-major, M = 128, N = 256.
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                            (static_cast<uint32_t>(BM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     ptx::smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ float tf32_head(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(g), "r"(bytes) : "memory");
}

/// MT: 128-row halves per CTA (1: 128 x 256 tiles, two CTAs per SM; 2: 256 x
/// 256 tiles, both TMEM accumulators, one CTA per SM, half the B traffic).
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

/// MCAST: launched as clusters of two CTAs along M that share each stage's B:
/// rank r copies half r (hi or lo) of the block and multicasts it to both,
/// halving the L2 reads of B (the GEMM's largest traffic).
template <int MT, bool MCAST = false>
__global__ void __launch_bounds__(kThreads * MT, MT == 1 ? 2 : 1)
tc_sgemm3_kernel(const float* __restrict__ A, int lda, const float* __restrict__ bt_hi,
                 const float* __restrict__ bt_lo, int ldb, float* __restrict__ C, std::size_t ldc, std::size_t M,
                 int N, int K, int* flag, const int* __restrict__ col_map, const int* __restrict__ a_map,
                 const float* __restrict__ fold_add, std::size_t ld_add, const float* __restrict__ b_sw,
                 int debug, int nfirst) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment of the swizzle atoms
    const uint32_t raw = ptx::smem_addr(smem_raw);
    unsigned char* base = smem_raw + ((1024 - (raw & 1023)) & 1023);
    constexpr int kAB = MT * kABytes;                  // A hi (or lo) per stage
    constexpr int kSB = 2 * kAB + 2 * kBBytes;          // stage bytes
    constexpr int kT = kThreads * MT;
    uint64_t* bar = reinterpret_cast<uint64_t*>(base + kStages * kSB); // one per stage: MMAs done
    uint64_t* bfull = bar + kStages;                                            // one per stage: B landed (TMA)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + kStages);
    const uint32_t sbase = ptx::smem_addr(base);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // nfirst: grid x = column tile, so the CTAs sharing an A row tile run
    // together (A leaves DRAM once; B, 2 MB, stays in L2 either way)
    const unsigned mi = nfirst ? blockIdx.y : blockIdx.x, ni = nfirst ? blockIdx.x : blockIdx.y;
    const std::size_t m0 = static_cast<std::size_t>(mi) * (BM * MT);
    const int n0 = static_cast<int>(ni) * BN;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         ptx::smem_addr(tmem_slot)),
                     "n"(kTmemCols * MT)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) {
            ptx::mbar_init(bar + i, 1);
            ptx::mbar_init(bfull + i, 1);
        }
        ptx::fence_mbar_init();
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    uint32_t crank = 0;
    if constexpr (MCAST) {
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
        cluster_sync_all(); // the peer's barriers exist before any multicast lands
    }

    // stage st: A hi, A lo, B hi, B lo.  A is fetched into registers one
    // chunk ahead (its global latency hides behind the barrier and the MMA
    // issue), then split and stored; B goes straight in by cp.async.
    constexpr int kAV = BM * MT * (BK / 4) / kT; // float4 of A per thread per chunk
    float4 areg[kAV];
    auto fetch_a = [&](int ch) {
        const int k0 = ch * BK;
#pragma unroll
        for (int u = 0; u < kAV; ++u) {
            const int i = tid + u * kT, r = i >> 2, c = i & 3, k = k0 + 4 * c;
            if (a_map) { // gathered columns (the folded inverse's W slots)
                const float* row = A + (m0 + r) * lda;
                const bool ok = m0 + r < M;
                areg[u] = make_float4(ok && k < K ? row[__ldg(a_map + k)] : 0.f,
                                      ok && k + 1 < K ? row[__ldg(a_map + k + 1)] : 0.f,
                                      ok && k + 2 < K ? row[__ldg(a_map + k + 2)] : 0.f,
                                      ok && k + 3 < K ? row[__ldg(a_map + k + 3)] : 0.f);
            } else {
                areg[u] = (m0 + r < M && k < K) ? *reinterpret_cast<const float4*>(A + (m0 + r) * lda + k)
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    };
    auto store_a = [&](int st) {
        unsigned char* g0 = base + st * kSB;
#pragma unroll
        for (int u = 0; u < kAV; ++u) {
            const int i = tid + u * kT, r = i >> 2, c = i & 3;
            const float4 v = areg[u];
            const float4 h = make_float4(tf32_head(v.x), tf32_head(v.y), tf32_head(v.z), tf32_head(v.w));
            const float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
            *reinterpret_cast<float4*>(g0 + sw64(r, c)) = h;
            *reinterpret_cast<float4*>(g0 + kAB + sw64(r, c)) = l;
        }
    };
    const int kblocks = (K + BK - 1) / BK;
    auto load_b = [&](int ch, int st) {
        if (MCAST) { // half of the block from each CTA of the pair, to both
            if (tid == 0) {
                ptx::mbar_expect_tx(bfull + st, 2 * kBBytes);
                const float* src = b_sw + (static_cast<std::size_t>(ni) * kblocks + ch) * (2 * BN * BK) +
                                   crank * (BN * BK);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], "
                    "%2, [%3], %4;\n" ::"r"(ptx::smem_addr(base + st * kSB + 2 * kAB + crank * kBBytes)),
                    "l"(src), "r"(static_cast<uint32_t>(kBBytes)), "r"(ptx::smem_addr(bfull + st)),
                    "h"(static_cast<uint16_t>(0x3))
                    : "memory");
            }
            return;
        }
        if (b_sw) { // pre-swizzled on the host: the stage's B (hi, lo) is one contiguous 32 KB block
            if (tid == 0) {
                ptx::mbar_expect_tx(bfull + st, 2 * kBBytes);
                ptx::bulk_load(base + st * kSB + 2 * kAB,
                               b_sw + (static_cast<std::size_t>(ni) * kblocks + ch) * (2 * BN * BK),
                               2 * kBBytes, bfull + st);
            }
            return;
        }
        const int k0 = ch * BK;
        const uint32_t s0 = sbase + st * kSB;
        for (int i = tid; i < BN * (BK / 4); i += kT) {
            const int r = i >> 2, c = i & 3, n = n0 + r, k = k0 + 4 * c;
            const int bytes = (n < N && k < K) ? 16 : 0;
            const std::size_t off = bytes ? static_cast<std::size_t>(n) * ldb + k : 0;
            cp_async16(s0 + 2 * kAB + sw64(r, c), bt_hi + off, bytes);
            cp_async16(s0 + 2 * kAB + kBBytes + sw64(r, c), bt_lo + off, bytes);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    const int nchunks = (K + BK - 1) / BK;
    uint32_t phases = 0u; // bit st: parity of stage st's next MMA completion
    fetch_a(0);
    load_b(0, 0);
    store_a(0);
    for (int ch = 0; ch < nchunks; ++ch) {
        const int st = ch % kStages;
        if (ch + 1 < nchunks) fetch_a(ch + 1);
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        ptx::fence_proxy_async(); // generic-proxy smem writes -> visible to the tensor core
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (tid == 0 && (debug & 2)) { // development knob: loads only, no MMAs
            if (b_sw || MCAST) ptx::mbar_wait(bfull + st, static_cast<uint32_t>((ch / kStages) & 1));
            ptx::mbar_arrive(bar + st);
        } else if (tid == 0) {
            if (b_sw || MCAST) ptx::mbar_wait(bfull + st, static_cast<uint32_t>((ch / kStages) & 1));
            const uint32_t s0 = sbase + st * kSB;
            const uint32_t bh = s0 + 2 * kAB, bl = s0 + 2 * kAB + kBBytes;
#pragma unroll
            for (int h = 0; h < MT; ++h) { // 128-row half h: rows 128 h.. of the A tile, accumulator h
                const uint32_t ah = s0 + h * kABytes, al = s0 + kAB + h * kABytes;
                const uint32_t td = tmem + static_cast<uint32_t>(h * BN);
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) { // 8 tf32 = 32 bytes per MMA step along K
                    const uint32_t o = 32u * kk;
                    const uint32_t acc0 = (ch > 0 || kk > 0) ? 1u : 0u;
                    mma_tf32(td, smem_desc(ah + o), smem_desc(bh + o), acc0);
                    mma_tf32(td, smem_desc(ah + o), smem_desc(bl + o), 1u);
                    mma_tf32(td, smem_desc(al + o), smem_desc(bh + o), 1u);
                }
            }
            mma_commit(bar + st);
        }
        if (ch + 1 < nchunks) {
            const int nx = (ch + 1) % kStages;
            if (ch + 1 >= kStages) { // the MMAs of chunk ch + 1 - kStages read that stage
                ptx::mbar_wait(bar + nx, (phases >> nx) & 1u);
                phases ^= 1u << nx;
                if constexpr (MCAST) cluster_sync_all(); // ... in both CTAs of the pair
            }
            load_b(ch + 1, nx);
            store_a(nx); // overlaps the MMAs of chunk ch
        }
    }
    // the last chunk's commit covers every earlier MMA of this thread
    {
        const int st = (nchunks - 1) % kStages;
        ptx::mbar_wait(bar + st, (phases >> st) & 1u);
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    bool bad = false;

    // epilogue: warp w owns TMEM lanes (= tile rows) 32w .. 32w + 31; the
    // stage buffers are free (every MMA has completed)
    if constexpr (MCAST) cluster_sync_all(); // no multicast into this CTA is still pending
    if (debug & 1) { // development knob: no epilogue
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();
        if (warp == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols * MT)
                         : "memory");
        return;
    }
    const int quarter = warp & 3, half = warp >> 2; // TMEM lane quarter, accumulator
    const std::size_t row = m0 + 128 * half + 32 * quarter + lane;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        const uint32_t taddr =
            tmem + (static_cast<uint32_t>(32 * quarter) << 16) + static_cast<uint32_t>(half * BN + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        const int n = n0 + c0;
        if (n == 0 && row < M) bad |= !isfinite(__uint_as_float(v[0])); // the DC coefficient
        // transpose through shared memory (this warp's 4 KB, 16-byte chunks
        // XOR-swizzled by row: conflict-free both ways), then each quarter-warp
        // stores one row's 128 contiguous bytes
        unsigned char* tb = base + warp * 4096;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            *reinterpret_cast<uint4*>(tb + lane * 128 + ((q ^ (lane & 7)) << 4)) =
                make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 8; ++it) {
            const int r = 4 * it + (lane >> 3), q = lane & 7;
            const uint4 w = *reinterpret_cast<const uint4*>(tb + r * 128 + ((q ^ (r & 7)) << 4));
            const std::size_t grow = m0 + 128 * half + 32 * quarter + r;
            const int col = n + 4 * q;
            if (grow < M && fold_add) { // unfold: x_c = w_c + v_c, x_{2N-1-c} = w_c - v_c
                const uint32_t e[4] = {w.x, w.y, w.z, w.w};
                const float* add = fold_add + grow * ld_add;
                float* orow = C + grow * ldc;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (col + u < N) {
                        const float wv = add[col + u], v = __uint_as_float(e[u]);
                        orow[col + u] = wv + v;
                        orow[2 * N - 1 - (col + u)] = wv - v;
                    }
            } else if (grow < M && col_map) { // scattered output columns (the folded route's slots)
                const uint32_t e[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (col + u < N) C[grow * ldc + __ldg(col_map + col + u)] = __uint_as_float(e[u]);
            } else if (grow < M) {
                float* dst = C + grow * ldc + col;
                if (col + 4 <= N) {
                    __stcs(reinterpret_cast<float4*>(dst), make_float4(__uint_as_float(w.x), __uint_as_float(w.y),
                                                                       __uint_as_float(w.z), __uint_as_float(w.w)));
                } else {
                    const uint32_t e[4] = {w.x, w.y, w.z, w.w};
                    for (int u = 0; u < 4 && col + u < N; ++u) dst[u] = __uint_as_float(e[u]);
                }
            }
        }
        __syncwarp();
    }
    if (bad) atomicOr(flag, 1);
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols * MT)
                     : "memory");
}

} // namespace

std::vector<float> tc_swizzle_b(const float* bt_hi, const float* bt_lo, int N, int K, int ldb) {
    const int ntiles = (N + BN - 1) / BN, kblocks = (K + BK - 1) / BK;
    std::vector<float> out(static_cast<std::size_t>(ntiles) * kblocks * 2 * BN * BK, 0.f);
    for (int nt = 0; nt < ntiles; ++nt)
        for (int kb = 0; kb < kblocks; ++kb) {
            float* blk = out.data() + (static_cast<std::size_t>(nt) * kblocks + kb) * (2 * BN * BK);
            for (int r = 0; r < BN; ++r)
                for (int kl = 0; kl < BK; ++kl) {
                    const int n = nt * BN + r, k = kb * BK + kl, c = kl >> 2;
                    const int at = (r * 64 + ((c ^ ((r >> 1) & 3)) << 4)) / 4 + (kl & 3);
                    if (n < N && k < K) {
                        blk[at] = bt_hi[static_cast<std::size_t>(n) * ldb + k];
                        blk[BN * BK + at] = bt_lo[static_cast<std::size_t>(n) * ldb + k];
                    }
                }
        }
    return out;
}

bool tc_sgemm3_supported(int K, int N, int lda, int ldb, std::size_t ldc, const void* A, const void* Bh,
                         const void* Bl, const void* C) {
    const auto al = [](const void* p) { return reinterpret_cast<std::uintptr_t>(p) % 16 == 0; };
    return K > 0 && N > 0 && K % 4 == 0 && lda % 4 == 0 && ldb % 4 == 0 && ldc % 4 == 0 && al(A) && al(Bh) &&
           al(Bl) && al(C);  // (with an A column map only the B and C constraints matter, and they are checked)
}

cudaError_t tc_sgemm3(const float* A, int lda, const float* bt_hi, const float* bt_lo, int ldb, float* C,
                      std::size_t ldc, std::size_t M, int N, int K, int* flag, cudaStream_t stream,
                      const int* col_map, const int* a_map, const float* fold_add, std::size_t ld_add,
                      const float* b_sw) {
    if (M == 0 || N == 0) return cudaSuccess;
    static const bool bulk_off = [] {
        const char* e = std::getenv("DCTP_TC32_BULK");
        return e && e[0] == '0';
    }();
    if (bulk_off) b_sw = nullptr;
    static const int debug = [] { // DCTP_TC32_DEBUG: 1 = skip the epilogue, 2 = skip the MMAs (timing only)
        const char* e = std::getenv("DCTP_TC32_DEBUG");
        return e ? std::atoi(e) : 0;
    }();
    static const int mt = [] {
        const char* e = std::getenv("DCTP_TC32_M256");
        return (e && e[0] == '1') ? 2 : 1;
    }();
    constexpr int kSmem2 = kStages * (4 * kABytes + 2 * kBBytes) + 1024 + 64;
    const cudaError_t attr1 = smem_optin(reinterpret_cast<const void*>(tc_sgemm3_kernel<1>), kSmem);
    const cudaError_t attr2 = smem_optin(reinterpret_cast<const void*>(tc_sgemm3_kernel<2>), kSmem2);
    if (attr1 != cudaSuccess) return attr1;
    if (attr2 != cudaSuccess) return attr2;
    static const bool mcast = [] { // opt-in: measured slower (the per-chunk cluster barrier)
        const char* e = std::getenv("DCTP_TC32_MCAST");
        return e && e[0] == '1';
    }();
    if (mcast && mt == 1 && b_sw) {
        const cudaError_t attr3 = smem_optin(reinterpret_cast<const void*>(tc_sgemm3_kernel<1, true>), kSmem);
        if (attr3 != cudaSuccess) return attr3;
        const unsigned gx = static_cast<unsigned>(((M + BM - 1) / BM + 1) / 2 * 2); // whole CTA pairs
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(gx, static_cast<unsigned>((N + BN - 1) / BN));
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = kSmem;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, tc_sgemm3_kernel<1, true>, A, lda, bt_hi, bt_lo, ldb, C, ldc, M, N, K, flag,
                                  col_map, a_map, fold_add, ld_add, b_sw, debug, 0);
    }
    static const int nfirst = [] {
        const char* e = std::getenv("DCTP_TC32_NFIRST");
        return (e && e[0] == '0') ? 0 : 1;
    }();
    const std::size_t rows_per_tile = static_cast<std::size_t>(BM) * mt;
    const std::size_t gm_all = (M + rows_per_tile - 1) / rows_per_tile;
    const unsigned gn = static_cast<unsigned>((N + BN - 1) / BN);
    // row tiles on grid.y (nfirst) are limited to 65535: launch row slices
    // (DCTP_TC32_SLICE_TILES lowers the slice for the tests)
    static const std::size_t slice = [] {
        const char* e = std::getenv("DCTP_TC32_SLICE_TILES");
        const long v = e ? std::atol(e) : 65535;
        return static_cast<std::size_t>(v >= 1 && v <= 65535 ? v : 65535);
    }();
    for (std::size_t t0 = 0; t0 < gm_all; t0 += slice) {
        const unsigned gm = static_cast<unsigned>(gm_all - t0 < slice ? gm_all - t0 : slice);
        const std::size_t r0 = t0 * rows_per_tile;
        const dim3 grid = nfirst ? dim3(gn, gm) : dim3(gm, gn);
        (mt == 2 ? tc_sgemm3_kernel<2> : tc_sgemm3_kernel<1>)<<<grid, kThreads * mt, mt == 2 ? kSmem2 : kSmem,
                                                               stream>>>(
            A + r0 * static_cast<std::size_t>(lda), lda, bt_hi, bt_lo, ldb, C + r0 * ldc, ldc, M - r0, N, K, flag,
            col_map, a_map, fold_add ? fold_add + r0 * ld_add : nullptr, ld_add, b_sw, debug, nfirst);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

} // namespace dctp::dev
