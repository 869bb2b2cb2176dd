// fp64 / smem latency microbenchmark (one warp, dependent chains).
#include <cstdio>
__global__ void lat(double* out, long long* cyc, int iters, double a, double b) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = i;
    __syncwarp();
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = x + a; x = x + b; x = x + a; x = x + b; }
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) { x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); }
    long long t2 = clock64();
    int idx = threadIdx.x;
    for (int i = 0; i < iters; ++i) { idx = (int)sm[idx & 1023]; idx = (int)sm[(idx + 1) & 1023]; idx = (int)sm[(idx + 2) & 1023]; idx = (int)sm[(idx+3) & 1023]; }
    long long t3 = clock64();
    float y = threadIdx.x;
    for (int i = 0; i < iters; ++i) { y = fmaf(y, (float)a, (float)b); y = fmaf(y, (float)a, (float)b); y = fmaf(y, (float)a, (float)b); y = fmaf(y, (float)a, (float)b); }
    long long t4 = clock64();
    out[threadIdx.x] = x + idx + y;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
    double* out; long long* cyc; cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 64);
    const int iters = 4096;
    lat<<<1, 32>>>(out, cyc, iters, 1.0000001, 1e-9);
    lat<<<1, 32>>>(out, cyc, iters, 1.0000001, 1e-9);
    long long h[4]; cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
    printf("{\"dadd_latency\": %.1f, \"dfma_latency\": %.1f, \"lds_dep_latency\": %.1f, \"ffma_latency\": %.1f}\n",
           h[0] / (4.0 * iters), h[1] / (4.0 * iters), h[2] / (4.0 * iters), h[3] / (4.0 * iters));
    return 0;
}
