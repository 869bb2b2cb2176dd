// tcgen05 peak probe (the denominators of the 3xTF32 GEMM's and the int8
// Ozaki GEMM's rooflines): every CTA issues back-to-back 128 x N x K MMAs from
// shared-memory operands into TMEM, one elected thread, a commit every 64
// MMAs; 148 x 2 CTAs; CUDA events around the launch.  Kinds: kind::tf32
// (N = 256, K = 8) and kind::i8 (N = 256 and N = 96 — the Ozaki kernel's
// tile — K = 32).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_peak tools/tc_peak.cu && tools/tc_peak
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t desc64(uint32_t a) { // K-major SWIZZLE_64B, SBO 512
    return static_cast<uint64_t>((a & 0x3FFFF) >> 4) | (1ull << 16) | (static_cast<uint64_t>(512 >> 4) << 32) |
           (1ull << 46) | (4ull << 61);
}

constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
template <int N>
__host__ __device__ constexpr uint32_t idesc_i8() { return (2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((128u >> 4) << 24); }

template <int KIND, int N> // KIND 0: tf32, 1: i8
__global__ void __launch_bounds__(128, 2) tc_peak_kernel(int iters, int* sink) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (8192 + 16384) / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(saddr(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(saddr(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint64_t a = desc64(saddr(smem)), b = desc64(saddr(smem + 8192));
        uint32_t phase = 0;
        for (int it = 0; it < iters; ++it) {
            if constexpr (KIND == 0)
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(a), "l"(b), "r"(kIdesc), "r"(it > 0 ? 1 : 0));
            else
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(a), "l"(b), "r"(idesc_i8<N>()), "r"(it > 0 ? 1 : 0));
            if ((it & 63) == 63 || it == iters - 1) {
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                                 saddr(&bar))
                             : "memory");
                asm volatile(
                    "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                        saddr(&bar)),
                    "r"(phase)
                    : "memory");
                phase ^= 1u;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tmem));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        if (v == 0x7fffffffu) atomicAdd(sink, 1);
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
    }
}

template <int KIND, int N>
double run(int sms, int* sink) {
    const int smem = 8192 + 16384;
    cudaFuncSetAttribute(tc_peak_kernel<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 20000, grid = 2 * sms;
    tc_peak_kernel<KIND, N><<<grid, 128, smem>>>(1000, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        tc_peak_kernel<KIND, N><<<grid, 128, smem>>>(iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    const double k = KIND == 0 ? 8 : 32;
    return 2.0 * 128 * N * k * static_cast<double>(iters) * grid / (best * 1e-3) / 1e12;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int* sink;
    cudaMalloc(&sink, sizeof(int));
    const double tf = run<0, 256>(sms, sink);
    const double i8 = run<1, 256>(sms, sink);
    const double i8n96 = run<1, 96>(sms, sink);
    std::printf("{\"tcgen05_tf32_tflops\": %.1f, \"tcgen05_i8_tops\": %.1f, \"tcgen05_i8_n96_tops\": %.1f, "
                "\"status\": \"%s\", \"how\": \"tools/tc_peak.cu: %d CTAs x 20000 back-to-back 128xNxK MMAs from "
                "shared memory (tf32 N=256 K=8; i8 N=256 and N=96, K=32), best of 5\"}\n",
                tf, i8, i8n96, cudaGetErrorString(cudaGetLastError()), 2 * sms);
    return 0;
}
