// HBM bandwidth by direction on the box: pure streaming writes (the output
// stream of the progressive / folded kernels), pure reads, and a copy —
// float4 accesses, grid = 148 x 8 CTAs x 256 threads, grid-stride; mean of
// 10 launches after warm-up, CUDA events.  Writes both plain and .cs
// (streaming) stores.  usage: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/hbm_rw.cu -o tools/hbm_rw && tools/hbm_rw
#include <cstdio>
#include <string>
#include <cuda_runtime.h>

__global__ void wr(float4* __restrict__ p, size_t n4, int cs) {
    const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        if (cs) __stcs(p + i, v); else p[i] = v;
}
__global__ void rd(const float4* __restrict__ p, size_t n4, float* sink) {
    float a = 0.f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 v = __ldcs(p + i);
        a += v.x + v.y + v.z + v.w;
    }
    if (a == 12345.f) *sink = a;
}
__global__ void cp(const float4* __restrict__ s, float4* __restrict__ d, size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        __stcs(d + i, __ldcs(s + i));
}

// C4's output pattern: 128-row x 256-column fp32 tiles of a [rows][2176]
// matrix, one CTA per tile, column tile slowest across the grid (the
// progressive GEMM's order) or fastest.
__global__ void tile_wr(float* __restrict__ c, size_t rows, int cols, int ntn, int nfast) {
    const size_t t = blockIdx.x;
    const size_t ntm = rows / 128;
    const size_t mt = nfast ? t / ntn : t % ntm, nt = nfast ? t % ntn : t / ntm;
    const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
    for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
        const int r = i / 64, c4 = i % 64;
        const size_t col = nt * 256 + 4 * c4;
        if (col < (size_t)cols) __stcs(reinterpret_cast<float4*>(c + (mt * 128 + r) * cols + col), v);
    }
}

// The same tiles from a persistent grid (one CTA per SM, tile range per
// CTA like the GEMM), `warps` storing warps per CTA.
__global__ void tile_wr_persist(float* __restrict__ c, size_t rows, int cols, int ntn) {
    const size_t ntm = rows / 128, total = ntm * ntn;
    const size_t first = total * blockIdx.x / gridDim.x, last = total * (blockIdx.x + 1) / gridDim.x;
    const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
    for (size_t t = first; t < last; ++t) {
        const size_t mt = t % ntm, nt = t / ntm;
        for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
            const int r = i / 64, c4 = i % 64;
            const size_t col = nt * 256 + 4 * c4;
            if (col < (size_t)cols) __stcs(reinterpret_cast<float4*>(c + (mt * 128 + r) * cols + col), v);
        }
    }
}

__global__ void tile_wr_strided(float* __restrict__ c, size_t rows, int cols, int ntn) {
    const size_t ntm = rows / 128, total = ntm * ntn;
    const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
    for (size_t t = blockIdx.x; t < total; t += gridDim.x) {
        const size_t mt = t % ntm, nt = t / ntm;
        for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
            const int r = i / 64, c4 = i % 64;
            const size_t col = nt * 256 + 4 * c4;
            if (col < (size_t)cols) __stcs(reinterpret_cast<float4*>(c + (mt * 128 + r) * cols + col), v);
        }
    }
}

int main() {
    const size_t bytes = 1ull << 30, n4 = bytes / 16;
    float4 *a, *b;
    float* sink;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(a, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = 148 * 8, threads = 256;
    auto run = [&](const char* name, double moved, auto&& f) {
        for (int i = 0; i < 3; ++i) f();
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"op\": \"%s\", \"GBps\": %.1f}\n", name, moved / (ms / 10 * 1e-3) / 1e9);
    };
    run("write", bytes, [&] { wr<<<grid, threads>>>(a, n4, 0); });
    run("write_cs", bytes, [&] { wr<<<grid, threads>>>(a, n4, 1); });
    run("read", bytes, [&] { rd<<<grid, threads>>>(a, n4, sink); });
    run("copy", 2.0 * bytes, [&] { cp<<<grid, threads>>>(a, b, n4); });
    {
        const size_t rows = 65536;
        const int cols = 2176, ntn = 9;
        const double moved = double(rows) * cols * 4;
        run("c4_tiles_colmajor", moved, [&] { tile_wr<<<(rows / 128) * ntn, 256>>>((float*)a, rows, cols, ntn, 0); });
        run("c4_tiles_rowmajor", moved, [&] { tile_wr<<<(rows / 128) * ntn, 256>>>((float*)a, rows, cols, ntn, 1); });
        for (int w : {8, 16})
            run((std::string("c4_tiles_strided_warps") + std::to_string(w)).c_str(), moved,
                [&] { tile_wr_strided<<<148, 32 * w>>>((float*)a, rows, cols, ntn); });
        for (int w : {4, 8, 16, 32})
            run((std::string("c4_tiles_persistent_warps") + std::to_string(w)).c_str(), moved,
                [&] { tile_wr_persist<<<148, 32 * w>>>((float*)a, rows, cols, ntn); });
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
