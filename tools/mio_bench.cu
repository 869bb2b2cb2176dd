// Shared-memory / shuffle throughput per SM on B200 (MIO pipe), with integer
// LOP3 accumulation so the fp64 pipe is not the limiter.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/mio_bench.cu -o tools/mio_bench
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

template <int MODE>
__global__ void k(unsigned* out) {
    __shared__ __align__(16) unsigned sm[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 2654435761u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned a0 = threadIdx.x, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll 8
    for (int it = 0; it < ITERS; ++it) {
        const int base = (it * 128) & 4095;
        if (MODE == 0) { // LDS.32 x4, consecutive lanes
            a0 ^= sm[base + lane]; a1 ^= sm[base + 32 + lane]; a2 ^= sm[base + 64 + lane]; a3 ^= sm[base + 96 + lane];
        } else if (MODE == 1) { // LDS.64 x2 (256 B per instr)
            const uint2 v = reinterpret_cast<const uint2*>(sm)[(base >> 1) + lane];
            const uint2 w = reinterpret_cast<const uint2*>(sm)[(base >> 1) + 32 + lane];
            a0 ^= v.x ^ w.x; a1 ^= v.y ^ w.y;
        } else if (MODE == 2) { // LDS.128 x1 (512 B per instr)
            const uint4 v = reinterpret_cast<const uint4*>(sm)[(base >> 2) + lane];
            a0 ^= v.x ^ v.y; a1 ^= v.z ^ v.w;
        } else if (MODE == 3) { // SHFL.32 x4
            a0 ^= __shfl_xor_sync(0xffffffffu, a1 + it, 1);
            a1 ^= __shfl_xor_sync(0xffffffffu, a2 + it, 2);
            a2 ^= __shfl_xor_sync(0xffffffffu, a3 + it, 4);
            a3 ^= __shfl_xor_sync(0xffffffffu, a0 + it, 8);
        } else if (MODE == 4) { // STS.64 x2
            reinterpret_cast<uint2*>(sm)[(base >> 1) + lane] = make_uint2(a0 + it, a1);
            reinterpret_cast<uint2*>(sm)[(base >> 1) + 32 + lane] = make_uint2(a2, a3 + it);
        } else if (MODE == 5) { // STS.128 x1
            reinterpret_cast<uint4*>(sm)[(base >> 2) + lane] = make_uint4(a0 + it, a1, a2, a3);
        } else if (MODE == 6) { // LDS.64 at 16-byte lane stride (2 lanes per 32 B: half-used lines)
            const uint2 v = reinterpret_cast<const uint2*>(sm)[(base >> 1) + 2 * lane];
            const uint2 w = reinterpret_cast<const uint2*>(sm)[(base >> 1) + 2 * lane + 1];
            a0 ^= v.x ^ w.x; a1 ^= v.y ^ w.y;
        }
    }
    if ((a0 ^ a1 ^ a2 ^ a3) == 0x12345678u) out[threadIdx.x] = a0;
}

template <int MODE>
float run(int sms, unsigned* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<MODE><<<sms, 1024>>>(out);
    cudaEventRecord(e0);
    k<MODE><<<sms, 1024>>>(out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    unsigned* out;
    cudaMalloc(&out, 1 << 20);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double clk = 1.965e9, warp_iters = 32.0 * ITERS;
    const char* names[] = {"4x LDS.32", "2x LDS.64", "1x LDS.128", "4x SHFL.32", "2x STS.64", "1x STS.128",
                           "2x LDS.64 16B-stride"};
    float ms[7] = {run<0>(sms, out), run<1>(sms, out), run<2>(sms, out), run<3>(sms, out),
                   run<4>(sms, out), run<5>(sms, out), run<6>(sms, out)};
    for (int m = 0; m < 7; ++m)
        printf("%-22s %.3f ms -> %.2f SM cycles per warp-iteration\n", names[m], ms[m], ms[m] * 1e-3 * clk / warp_iters);
    return 0;
}
