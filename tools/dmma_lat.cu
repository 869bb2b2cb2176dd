// DMMA m8n8k4 latency (dependent chain, one warp) and per-SMSP throughput vs chains.
#include <cstdio>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void chains(double* out, long long* cyc, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[CH][2];
    for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
    long long t1 = clock64();
    double s = 0; for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int CH> void run(int warps) {
    double* out; long long* cyc; cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 8);
    int iters = 2048;
    chains<CH><<<1, 32 * warps>>>(out, cyc, iters);
    chains<CH><<<1, 32 * warps>>>(out, cyc, iters);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("chains/warp %d warps/CTA %2d (warps/SMSP %.1f): %.1f cycles per DMMA per warp-chain step; SM rate %.2f DMMA/cycle\n",
           CH, warps, warps / 4.0, (double)h / iters, (double)CH * warps * iters / h);
}
int main() {
    run<1>(1); run<2>(1); run<4>(1); run<8>(1);
    run<1>(4); run<4>(4); run<8>(4); run<4>(8); run<2>(8); run<8>(8); run<4>(16);
    return 0;
}
