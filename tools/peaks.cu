// Measures the arithmetic peaks the DCT+ roofline needs and MEASURED_PEAKS.json
// lacks: fp64 / fp32 FMA on the CUDA cores and fp64 MMA (DMMA) on the tensor
// cores.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/peaks.cu -o tools/peaks
// Output: one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

template <class T, int ILP>
__global__ void fma_loop(T* out, int iters, T a, T b) {
    T acc[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = static_cast<T>(threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
    }
    T s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += acc[i];
    if (s == static_cast<T>(-1.2345)) out[threadIdx.x] = s;
}

// packed fp32 FMA (FFMA2, sm_100): two FMAs per lane per instruction
__global__ void ffma2_loop(float* out, int iters) {
    unsigned long long acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float v = static_cast<float>(threadIdx.x + i);
        asm("mov.b64 %0, {%1, %2};" : "=l"(acc[i]) : "f"(v), "f"(v + 1.0f));
    }
    unsigned long long a, b;
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(1.0000001f), "f"(1.0000002f));
    asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(1e-7f), "f"(2e-7f));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(a), "l"(b));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[i]));
        s += lo + hi;
    }
    if (s == -1.2345f) out[threadIdx.x] = s;
}

// m8n8k4 f64: 256 FMA per warp instruction
__global__ void dmma_m8n8k4(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == -1.2345) out[threadIdx.x] = s;
}

// m16n8k16 f64: 2048 FMA per warp instruction
__global__ void dmma_m16n8k16(double* out, int iters) {
    double a[8], b[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
    double c[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
                "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                  "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == -1.2345) out[threadIdx.x] = s;
}

template <class F>
float time_ms(F&& launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 1 << 20);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    const double fma64 = time_ms([&] { fma_loop<double, 8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-7); });
    const double tf64 = 2.0 * blocks * threads * 8.0 * iters / (fma64 * 1e-3) / 1e12;
    const double fma32 =
        time_ms([&] { fma_loop<float, 8><<<blocks, threads>>>((float*)out, iters, 1.0000001f, 1e-7f); });
    const double tf32 = 2.0 * blocks * threads * 8.0 * iters / (fma32 * 1e-3) / 1e12;
    const double f2 = time_ms([&] { ffma2_loop<<<blocks, threads>>>((float*)out, iters); });
    const double tf32x2 = 2.0 * 2.0 * blocks * threads * 8.0 * iters / (f2 * 1e-3) / 1e12;
    const int diters = 1024;
    const double d1 = time_ms([&] { dmma_m8n8k4<<<blocks, threads>>>(out, diters); });
    const double tdm1 = 2.0 * 256.0 * 8 * (blocks * threads / 32.0) * diters / (d1 * 1e-3) / 1e12;
    const double d2 = time_ms([&] { dmma_m16n8k16<<<blocks, threads>>>(out, diters / 4); });
    const double tdm2 = 2.0 * 2048.0 * 4 * (blocks * threads / 32.0) * (diters / 4) / (d2 * 1e-3) / 1e12;
    cudaError_t e = cudaDeviceSynchronize();
    printf("{\"sms\": %d, \"clock_mhz_attr\": %d, \"fp64_fma_tflops\": %.2f, \"fp32_fma_tflops\": %.2f, "
           "\"fp32_ffma2_tflops\": %.2f, \"dmma_m8n8k4_tflops\": %.2f, \"dmma_m16n8k16_tflops\": %.2f, "
           "\"status\": \"%s\"}\n",
           sms, clk / 1000, tf64, tf32, tf32x2, tdm1, tdm2, cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
