// Checks the register layout assumed for mma.m16n8k16 .f64 against a CPU product:
//   A (16x16, row): a[i] = A[g + 8*(i%2)][t + 4*(i/2)],  i < 8
//   B (16x8, col):  b[j] = B[t + 4*j][g],                 j < 4
//   C/D (16x8):     d[i] = D[g + 8*(i/2)][2t + (i%2)],    i < 4
// (g = lane / 4, t = lane % 4).  Prints the max abs error.
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(const double* A, const double* B, double* D) {
    const int lane = threadIdx.x, g = lane / 4, t = lane % 4;
    double a[8], b[4], d[4] = {0, 0, 0, 0};
    for (int i = 0; i < 8; ++i) a[i] = A[(g + 8 * (i % 2)) * 16 + t + 4 * (i / 2)];
    for (int j = 0; j < 4; ++j) b[j] = B[(t + 4 * j) * 8 + g];
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
        "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
          "d"(b[1]), "d"(b[2]), "d"(b[3]));
    for (int i = 0; i < 4; ++i) D[(g + 8 * (i / 2)) * 8 + 2 * t + (i % 2)] = d[i];
}

int main() {
    double hA[256], hB[128], hD[128];
    for (int i = 0; i < 256; ++i) hA[i] = std::sin(1.0 + i * 0.37);
    for (int i = 0; i < 128; ++i) hB[i] = std::cos(2.0 + i * 0.11);
    double *A, *B, *D;
    cudaMalloc(&A, sizeof hA);
    cudaMalloc(&B, sizeof hB);
    cudaMalloc(&D, sizeof hD);
    cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(A, B, D);
    cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int r = 0; r < 16; ++r)
        for (int c = 0; c < 8; ++c) {
            double s = 0;
            for (int kk = 0; kk < 16; ++kk) s += hA[r * 16 + kk] * hB[kk * 8 + c];
            err = std::fmax(err, std::fabs(s - hD[r * 8 + c]));
        }
    printf("m16n8k16 f64 layout max abs error %.3e (%s)\n", err, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
