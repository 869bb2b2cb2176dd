// tcgen05 kind::i8 issue-rate probe at the Ozaki kernels' tile widths: one
// issuing thread per CTA (cta_group::1, M = 128, one CTA per SM) or per CTA
// pair (cta_group::2, M = 256, 74 clusters), A from shared memory or from TMEM
// ([a_tmem]), N in {64, 96, 128, 192, 256}, 4 / 4 / 3 / 2 / 1 round-robin
// accumulators (no MMA waits on the one just issued), commits every 64 MMAs
// with two groups in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_peak_pair tools/tc_peak_pair.cu && tools/tc_peak_pair
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t desc64(uint32_t a) { // K-major SWIZZLE_64B, SBO 512
    return static_cast<uint64_t>((a & 0x3FFFF) >> 4) | (1ull << 16) | (static_cast<uint64_t>(512 >> 4) << 32) |
           (1ull << 46) | (4ull << 61);
}

__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t parity) {
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                     saddr(bar)),
                 "r"(parity)
                 : "memory");
}

template <int CG, int N>
__host__ __device__ constexpr uint32_t idesc() {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | (((CG == 2 ? 256u : 128u) >> 4) << 24);
}

template <int CG, int ASRC, int N>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint32_t a_tmem, uint64_t b, uint32_t acc) {
    if constexpr (CG == 1 && ASRC == 0)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(d), "l"(a), "l"(b), "r"(idesc<CG, N>()), "r"(acc));
    else if constexpr (CG == 1)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc<CG, N>()), "r"(acc));
    else if constexpr (ASRC == 0)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(d), "l"(a), "l"(b), "r"(idesc<CG, N>()), "r"(acc));
    else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc<CG, N>()), "r"(acc));
}

template <int CG>
__device__ __forceinline__ void commit(uint64_t* bar) {
    if constexpr (CG == 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(saddr(bar))
                     : "memory");
    else
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                saddr(bar)),
            "h"(static_cast<uint16_t>(3))
            : "memory");
}

template <int CG, int ASRC, int N>
__global__ void __launch_bounds__(128, 1) probe(int iters, int* sink) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint64_t bars[2];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    uint32_t rank = 0;
    if constexpr (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (int i = threadIdx.x; i < (8192 + 16384) / 4; i += blockDim.x) reinterpret_cast<int*>(smem)[i] = 0;
    if (warp == 0) {
        if constexpr (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(saddr(&slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(saddr(&slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
        }
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(saddr(&bars[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(saddr(&bars[1])));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if constexpr (CG == 2)
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = slot, a_tmem = slot + 448;
    constexpr int kAcc = N <= 96 ? 4 : (N <= 128 ? 3 : (N <= 192 ? 2 : 1));
    uint32_t phase = 0; // bit j: parity of bars[j]
    const int groups = iters / 64;
    if (threadIdx.x == 0 && rank == 0) {
        const uint64_t a = desc64(saddr(smem)), b = desc64(saddr(smem + 8192));
        for (int k = 0; k < groups; ++k) { // 64 MMAs per group, unrolled (constant accumulator offsets)
#pragma unroll
            for (int i = 0; i < 64; ++i) mma<CG, ASRC, N>(tmem + (i % kAcc) * N, a, a_tmem, b, (k > 0 || i >= kAcc) ? 1u : 0u);
            commit<CG>(&bars[k & 1]); // then wait for group k - 1
            if (k > 0) {
                const int j = (k - 1) & 1;
                wait_bar(&bars[j], (phase >> j) & 1u);
                phase ^= 1u << j;
            }
        }
        const int j = (groups - 1) & 1;
        wait_bar(&bars[j], (phase >> j) & 1u);
    } else if (CG == 2 && threadIdx.x == 0) { // the peer follows the leader's commits
        for (int k = 0; k < groups; ++k) {
            const int j = k & 1;
            wait_bar(&bars[j], (phase >> j) & 1u);
            phase ^= 1u << j;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if constexpr (CG == 2)
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (warp == 0) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tmem));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        if (v == 0x7fffffffu) atomicAdd(sink, 1);
        if constexpr (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

template <int CG, int ASRC, int N>
double run(int sms, int* sink) {
    const int smem = 8192 + 16384;
    cudaFuncSetAttribute(probe<CG, ASRC, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 40960, grid = sms / 2 * 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, probe<CG, ASRC, N>, 1000, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        cudaLaunchKernelEx(&cfg, probe<CG, ASRC, N>, iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    return 2.0 * 128 * N * 32 * static_cast<double>(iters) * grid / (best * 1e-3) / 1e12;
}

template <int CG, int ASRC>
void row(const char* name, int sms, int* sink, bool last) {
    std::printf("\"%s\": {\"64\": %.1f, \"96\": %.1f, \"128\": %.1f, \"192\": %.1f, \"256\": %.1f}%s", name,
                run<CG, ASRC, 64>(sms, sink), run<CG, ASRC, 96>(sms, sink), run<CG, ASRC, 128>(sms, sink),
                run<CG, ASRC, 192>(sms, sink), run<CG, ASRC, 256>(sms, sink), last ? "" : ", ");
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int* sink;
    cudaMalloc(&sink, sizeof(int));
    std::printf("{");
    row<1, 0>("cta1_smem_a", sms, sink, false);
    row<1, 1>("cta1_tmem_a", sms, sink, false);
    row<2, 0>("pair_smem_a", sms, sink, false);
    row<2, 1>("pair_tmem_a", sms, sink, false);
    std::printf(", \"unit\": \"TOPS\", \"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
