// Shared-memory radix-8 FFT building blocks for the DCT kernels (dct.cu) and
// the NFST fast route (nfst.cu), sm_100a.
#pragma once

#include "kernels/common.cuh"

namespace dctp::dev {

/// Shared-memory layout of the FFT rows: one complex of padding after every
/// 8, so the strided groups of every pass (including the bit-reversed gather
/// of the first one) hit 8 distinct 16-byte bank groups per quarter-warp.
__device__ __forceinline__ int pad8(int i) { return i + (i >> 3); }
__host__ __device__ constexpr int padded_len(int N) { return N + (N >> 3) + 1; }

/// Q consecutive radix-2 DIT stages (s0+1 .. s0+Q) fused into one pass over
/// groups of 2^Q elements held in registers: group (block, j) holds elements
/// block*2^(s0+Q) + j + m*2^s0, m < 2^Q, of the bit-reversed sequence.  One
/// shared-memory round trip and one barrier per Q stages instead of per stage.
/// The first pass (FIRST, s0 = 0) gathers its inputs from the natural-order
/// buffer `src` at the bit-reversed positions and writes `dst`, so no
/// bit-reversed scatter is ever stored.  `tw` holds e^{-2 pi i k / (N 2^tw_extra)}:
/// a table built for a longer transform is read with stride 2^tw_extra.
template <class T, bool Inverse, int Q, bool FIRST>
__device__ __forceinline__ void dit_group_pass(const cplx_t<T>* src, cplx_t<T>* dst, int rows, int N, int logN,
                                               int s0, const T* __restrict__ tw, int tw_extra = 0) {
    constexpr int G = 1 << Q;
    const int h0 = 1 << s0;
    const int lg = logN - Q; // log2 of the groups per row
    const int ld = padded_len(N);
    for (int t = threadIdx.x; t < (rows << lg); t += blockDim.x) {
        const int row = t >> lg, g = t & ((1 << lg) - 1);
        const int j = g & (h0 - 1), base = (g >> s0) * (h0 << Q) + j;
        cplx_t<T> v[G];
#pragma unroll
        for (int m = 0; m < G; ++m)
            v[m] = FIRST ? src[row * ld + pad8(static_cast<int>(bit_reverse(static_cast<unsigned>(base + m), logN)))]
                         : dst[row * ld + pad8(base + m * h0)];
#pragma unroll
        for (int tt = 0; tt < Q; ++tt) {
            const int span = 1 << tt;
            const int shift = logN - (s0 + tt + 1) + tw_extra; // twiddle step N / (2 * half)
            // stage tt needs w_q = W^((j + q h0) 2^shift), q < span; since
            // h0 2^shift is a quarter turn's multiple, w_{q + span/2} = -i w_q
            // (conjugated for the inverse): exact, so only the first half of
            // each stage's twiddles is loaded
            cplx_t<T> w[G / 2];
#pragma unroll
            for (int q = 0; q < span; ++q) {
                if (span >= 2 && q >= span / 2) {
                    const cplx_t<T> u = w[q - span / 2];
                    w[q] = Inverse ? cplx_t<T>{-u.y, u.x} : cplx_t<T>{u.y, -u.x};
                } else {
                    const cplx_t<T> u = __ldg(reinterpret_cast<const cplx_t<T>*>(tw) + ((j + q * h0) << shift));
                    w[q] = {u.x, Inverse ? -u.y : u.y};
                }
            }
#pragma unroll
            for (int m = 0; m < G; ++m) {
                if (m & span) continue;
                const T wr = w[m & (span - 1)].x, wi = w[m & (span - 1)].y;
                const cplx_t<T> a = v[m], b = v[m + span];
                const T br = b.x * wr - b.y * wi, bi = b.x * wi + b.y * wr;
                v[m] = {a.x + br, a.y + bi};
                v[m + span] = {a.x - br, a.y - bi};
            }
        }
#pragma unroll
        for (int m = 0; m < G; ++m) dst[row * ld + pad8(base + m * h0)] = v[m];
    }
    __syncthreads();
}

/// FFT of `rows` rows of N = 2^logN points given in natural order in `src`
/// (padded rows), result in natural order in `dst`: a bit-reversed gather
/// folded into the first radix-8 pass, then in-place radix-8 DIT passes
/// (radix-4/2 for the remainder).  `src` is dead afterwards.
template <class T, bool Inverse>
__device__ __forceinline__ void fft_rows(const cplx_t<T>* src, cplx_t<T>* dst, int rows, int N, int logN,
                                         const T* __restrict__ tw, int tw_extra = 0) {
    if (logN == 0) {
        for (int r = threadIdx.x; r < rows; r += blockDim.x) dst[r * padded_len(N)] = src[r * padded_len(N)];
        __syncthreads();
        return;
    }
    const int q0 = min(3, logN);
    if (q0 == 3) dit_group_pass<T, Inverse, 3, true>(src, dst, rows, N, logN, 0, tw, tw_extra);
    if (q0 == 2) dit_group_pass<T, Inverse, 2, true>(src, dst, rows, N, logN, 0, tw, tw_extra);
    if (q0 == 1) dit_group_pass<T, Inverse, 1, true>(src, dst, rows, N, logN, 0, tw, tw_extra);
    int s0 = q0;
    for (; s0 + 3 <= logN; s0 += 3) dit_group_pass<T, Inverse, 3, false>(dst, dst, rows, N, logN, s0, tw, tw_extra);
    if (logN - s0 == 2) dit_group_pass<T, Inverse, 2, false>(dst, dst, rows, N, logN, s0, tw, tw_extra);
    if (logN - s0 == 1) dit_group_pass<T, Inverse, 1, false>(dst, dst, rows, N, logN, s0, tw, tw_extra);
}

/// In-place FFT of one padded row of N = 2^logN points whose producer
/// already stored element i at position bit_reverse(i) (no permutation pass):
/// the radix-8 DIT passes only; natural-order output.  The NFST kernels
/// (nfst.cu) use it for rows too long to keep a second buffer beside them
/// in shared memory (n = 8192: 8192 complex doubles = 144 KB padded).
template <class T, bool Inverse>
__device__ __forceinline__ void fft_from_bitreversed(cplx_t<T>* buf, int N, int logN, const T* __restrict__ tw,
                                                     int tw_extra = 0) {
    int s0 = 0;
    for (; s0 + 3 <= logN; s0 += 3) dit_group_pass<T, Inverse, 3, false>(buf, buf, 1, N, logN, s0, tw, tw_extra);
    if (logN - s0 == 2) dit_group_pass<T, Inverse, 2, false>(buf, buf, 1, N, logN, s0, tw, tw_extra);
    if (logN - s0 == 1) dit_group_pass<T, Inverse, 1, false>(buf, buf, 1, N, logN, s0, tw, tw_extra);
}

} // namespace dctp::dev
