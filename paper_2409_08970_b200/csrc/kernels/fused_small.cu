// Fused persistent forward DCT+ for small plans (power-of-two n <= 512, at
// most 128 kept DCT indices and 128 secular roots), fp64, sm_100a.
//
// Warp-specialised, one CTA per SM, four warpgroups:
//   producer (warpgroups 2-3): TMA 1-D bulk loads of signal tiles (double-
//     buffered, mbarrier completion) -> orthonormal DCT-II of every row in
//     shared memory (Makhoul packing fused into the first Stockham pass of an
//     n/2-point complex FFT with compile-time radix-2/4 passes and per-pass
//     twiddle tables; real split + e^{-i pi k/2n} rotation) -> uniform gathers:
//     kept coefficients into the A tile of the Cauchy product, pass-through
//     coefficients (signed) straight into their output slots
//     (fast_transform.hpp:171);
//   consumers (warpgroups 0-1): the Cauchy stage on the fp64 tensor cores
//     (mma.sync m8n8k4 DMMA), out[s, slot_c] = sum_k shat[s, kept_k] T[k, c],
//     T[k, c] = sigma_c a_c z_k / (lambda_k - mu_c) (the reference's dense T_r,
//     fast_transform.hpp:355-366, transposed) held in REGISTERS as m8n8k4 B
//     fragments for the whole kernel (K x A <= 128 x 128 fp64 over 8 warps),
//     then the epilogue writes the active slots and one consumer thread sends
//     the assembled tile out with a TMA 1-D bulk store.
// Producer and consumers run one tile apart, synchronised by mbarriers, so
// the DCT of tile i+1 overlaps the DMMA work of tile i.  HBM traffic is the
// algorithmic minimum: every signal is read once and every coefficient
// written once.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "kernels/common.cuh"
#include "kernels/launch.hpp"

namespace dctp::dev {
namespace {

constexpr int kProducerThreads = 256; // warpgroups 2-3: TMA + DCT (setmaxnreg 88)
constexpr int kConsumerWarps = 8;     // warpgroups 0-1: DMMA Cauchy stage (setmaxnreg 168)
constexpr int kThreads = kProducerThreads + 32 * kConsumerWarps;
constexpr int KTMAX = 32;          // k-tiles of 4: K <= 128
constexpr int LDA = KTMAX * 4 + 4; // A-tile row stride (doubles): +4 staggers the 8 fragment rows over banks

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

template <int R>
__device__ __forceinline__ void butterfly(double2 (&v)[R]);

template <>
__device__ __forceinline__ void butterfly<2>(double2 (&v)[2]) {
    const double2 a = v[0], b = v[1];
    v[0] = make_double2(a.x + b.x, a.y + b.y);
    v[1] = make_double2(a.x - b.x, a.y - b.y);
}

template <>
__device__ __forceinline__ void butterfly<4>(double2 (&v)[4]) {
    // forward radix-4 DFT (e^{-2 pi i / 4} = -i)
    const double2 a0 = make_double2(v[0].x + v[2].x, v[0].y + v[2].y);
    const double2 a1 = make_double2(v[0].x - v[2].x, v[0].y - v[2].y);
    const double2 a2 = make_double2(v[1].x + v[3].x, v[1].y + v[3].y);
    const double2 a3 = make_double2(v[1].y - v[3].y, v[3].x - v[1].x); // -i (v1 - v3)
    v[0] = make_double2(a0.x + a2.x, a0.y + a2.y);
    v[2] = make_double2(a0.x - a2.x, a0.y - a2.y);
    v[1] = make_double2(a1.x + a3.x, a1.y + a3.y);
    v[3] = make_double2(a1.x - a3.x, a1.y - a3.y);
}

__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 2, %0;\n" ::"n"(32 * kConsumerWarps) : "memory");
}

/// Stockham pass layout for an N-point FFT: the first pass is radix-2 when
/// log2 N is odd, every other pass radix-4.  Pass p has sub-transform size
/// NS = 2^lns_of(p) and radix_of(p); its twiddles e^{-2 pi i r jm/(NS R)}
/// (jm < NS, 1 <= r < R) live at twiddle_offset(p) in the per-pass table.
template <int N>
struct Passes {
    static constexpr int LOG = __builtin_ctz(N);
    static constexpr int FIRST_R = (LOG % 2) ? 2 : 4;
    static constexpr int COUNT = (LOG % 2) ? 1 + (LOG - 1) / 2 : LOG / 2;
    static constexpr int radix(int p) { return p == 0 ? FIRST_R : 4; }
    static constexpr int lns(int p) { return p == 0 ? 0 : (FIRST_R == 2 ? 1 : 2) + 2 * (p - 1); }
    static constexpr int twiddle_offset(int p) {
        int off = 0;
        for (int q = 1; q < p; ++q) off += (1 << lns(q)) * (radix(q) - 1);
        return off;
    }
    static constexpr int TWIDDLES = twiddle_offset(COUNT);
};

/// for (t = lane; t < TOTAL; t += 32) f(t), with a compile-time trip count.
template <int TOTAL, class F>
__device__ __forceinline__ void lane_loop(int lane, F&& f) {
#pragma unroll
    for (int i = 0; i < TOTAL / 32; ++i) f(lane + 32 * i);
    if constexpr (TOTAL % 32 != 0) {
        const int t = lane + 32 * (TOTAL / 32);
        if (t < TOTAL) f(t);
    }
}

/// One Stockham (autosort) pass (P >= 1) over the SPW signals one producer
/// warp owns; lanes stride over the butterflies, the SPW rows interleave.
template <int N, int SPW, int P>
__device__ __forceinline__ void stockham_pass(const double2* __restrict__ src, double2* __restrict__ dst,
                                              const double2* __restrict__ ptw, int lane) {
    constexpr int R = Passes<N>::radix(P), LNS = Passes<N>::lns(P), NS = 1 << LNS;
    constexpr int M = N / R;
    constexpr int TWO = Passes<N>::twiddle_offset(P);
    lane_loop<SPW * M>(lane, [&](int t) {
        const int sig = t / M, j = t % M;
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = src[sig * N + j + r * M];
        const int jm = j & (NS - 1);
#pragma unroll
        for (int r = 1; r < R; ++r) v[r] = cmul(v[r], ptw[TWO + jm * (R - 1) + (r - 1)]);
        butterfly<R>(v);
        const int d = (j >> LNS) * (NS * R) + jm;
#pragma unroll
        for (int r = 0; r < R; ++r) dst[sig * N + d + r * NS] = v[r];
    });
}

/// Pass 0 straight from the real signal rows.  Makhoul's packing
/// w_m = v_{2m} + i v_{2m+1}, v = (x0, x2, ..., x3, x1), means every block of
/// four samples x[4b..4b+3] (b < N/2) holds w_b = (x[4b], x[4b+2]) and
/// w_{N-1-b} = (x[4b+3], x[4b+1]).  Butterflies j and j' = M-1-j of a radix-R
/// pass (M = N/R) together need exactly the blocks j + rM and j' + rM for
/// r < R/2, so each task loads R contiguous 32-byte blocks and runs both.
template <int N, int SPW>
__device__ __forceinline__ void stockham_first(const double* __restrict__ x, double2* __restrict__ dst, int lane,
                                               int valid_rows, bool& bad) {
    constexpr int R = Passes<N>::FIRST_R, M = N / R, n = 2 * N;
    (void)valid_rows;
    (void)bad;
    lane_loop<SPW * (M / 2)>(lane, [&](int t) {
        const int sig = t / (M / 2), j = t % (M / 2), jp = M - 1 - j;
        const double* xr = x + sig * n;
        double2 a[R], c[R]; // butterflies j and j'
#pragma unroll
        for (int r = 0; r < R / 2; ++r) {
            const double2 b0 = *reinterpret_cast<const double2*>(xr + 4 * (j + r * M));
            const double2 b1 = *reinterpret_cast<const double2*>(xr + 4 * (j + r * M) + 2);
            const double2 e0 = *reinterpret_cast<const double2*>(xr + 4 * (jp + r * M));
            const double2 e1 = *reinterpret_cast<const double2*>(xr + 4 * (jp + r * M) + 2);
            a[r] = make_double2(b0.x, b1.x);
            c[R - 1 - r] = make_double2(b1.y, b0.y);
            c[r] = make_double2(e0.x, e1.x);
            a[R - 1 - r] = make_double2(e1.y, e0.y);
        }
        butterfly<R>(a);
        butterfly<R>(c);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            dst[sig * N + j * R + r] = a[r];
            dst[sig * N + jp * R + r] = c[r];
        }
    });
}

/// Runs passes P.. of the FFT for one warp's rows, ping-ponging between a and
/// b (warp-synchronous: no CTA barrier); returns the buffer with the result.
template <int N, int SPW, int P>
__device__ __forceinline__ double2* fft_passes(double2* a, double2* b, const double2* ptw, int lane) {
    if constexpr (P == Passes<N>::COUNT) {
        return a; // `a` holds the output of the last pass
    } else {
        stockham_pass<N, SPW, P>(a, b, ptw, lane);
        __syncwarp();
        return fft_passes<N, SPW, P + 1>(b, a, ptw, lane);
    }
}

/// FOLD = false: generic plan, the DCT has length L = n.
/// FOLD = true : antisymmetric update (every kept DCT index is odd).  Then
///   shat_{2m+1} = sqrt(2/n) sum_j u_j cos(pi (2m+1)(2j+1)/2n),  u_j = x_j - x_{n-1-j},
///   shat_{2m}   = DCT-II_{n/2}(y)_m / sqrt(2),                y_j = x_j + x_{n-1-j},
/// so the Cauchy stage runs on u against W = D_odd^T T (the DCT-IV folded into
/// the plan's matrix, same DMMA work as T) and only the length-n/2 DCT-II of y
/// goes through the FFT — half the producer work (deflation).
/// The tile scheduler's counter pair re-arms itself: ctr[0] hands out tile
/// tickets, ctr[1] counts CTAs that have made their last claim; the last CTA
/// zeroes both, so the next launch on the same stream finds them at 0 without
/// a memset (a memset would queue behind the copy engines' PCIe transfers in
/// the host-buffer pipeline).  `last_ticket` is the CTA's final (prefetched)
/// claim: reading it makes sure that atomic has returned before the release.
__device__ __forceinline__ void release_counter(unsigned long long* ctr, long long last_ticket) {
    if (last_ticket < 0) return; // never: tickets are non-negative
    __threadfence();
    if (atomicAdd(ctr + 1, 1ull) == gridDim.x - 1) {
        ctr[0] = 0;
        ctr[1] = 0;
        __threadfence();
    }
}

template <int LOGN, int NTW, int KT, int TS, bool FOLD>
__global__ void __launch_bounds__(kThreads, 1)
fused_small_fwd_kernel(const double* __restrict__ in, double* __restrict__ out, std::size_t batch, SmallPlanDev P,
                       int* flag, unsigned long long* tile_counter) {
    constexpr int n = 1 << LOGN, L = FOLD ? n / 2 : n, NC = L / 2, MT = TS / 8;
    constexpr int TILE = TS * n; // doubles per signal tile
    using PS = Passes<NC>;
    extern __shared__ __align__(128) unsigned char smem[];
    double* xin = reinterpret_cast<double*>(smem);            // 2 x TILE: TMA-loaded input tiles
    double* xout = xin + 2 * TILE;                             // 2 x TILE: assembled output tiles
    double2* cw = reinterpret_cast<double2*>(xout + 2 * TILE); // TILE/2 complex: FFT ping-pong partner
    double* atile = reinterpret_cast<double*>(cw + TILE / 2);  // 2 x TS x LDA: Cauchy A operand
    double2* ptw = reinterpret_cast<double2*>(atile + 2 * TS * LDA);
    double2* sp = ptw + (PS::TWIDDLES > 0 ? PS::TWIDDLES : 1);
    double2* rt = sp + NC;
    double2* rt2 = rt + NC + 1;                          // rt * sqrt(2/L) / 2
    double* pass_coef = reinterpret_cast<double*>(rt2 + NC + 1); // n: sign (or sign/sqrt2 when folded)
    int* kept_idx = reinterpret_cast<int*>(pass_coef + n); // KT*4
    int* pass_src = kept_idx + 4 * KT;                     // n: index into the length-L coefficients
    int* pass_dst = pass_src + n;                          // n: output slot
    uint64_t* bars = reinterpret_cast<uint64_t*>(pass_dst + n);
    uint64_t* xfull = bars;       // [2] TMA load landed
    uint64_t* afull = bars + 2;   // [2] producer -> consumers: A tile + pass-through written
    uint64_t* aempty = bars + 4;  // [2] consumers -> producer: A tile consumed
    uint64_t* xofree = bars + 6;  // [2] output tile's TMA store has read it
    uint64_t* xempty = bars + 8;  // [2] every producer warp is done reading xin[b]
    // dynamic tile scheduler: the producer claims tiles from a global counter
    // (idle SMs take more work; static round-robin left a 40% tail)
    long long* sched = reinterpret_cast<long long*>(bars + 10);  // [2] tile landing in xin[b]
    long long* csched = sched + 2;                               // [2] tile whose A tile is in atile[b]

    const long long t_entry = clock64();
    unsigned long long g_entry;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_entry));
    const int tid = threadIdx.x;
    const int n_pass = P.n_pass;
    static_assert(kThreads == 512, "register split 256 x 88 + 256 x 168 assumes 512 threads");

    // ---- prologue: tables, barriers ---------------------------------------------
    {
        const double2* fft = reinterpret_cast<const double2*>(P.fft_tw);
#pragma unroll 1
        for (int p = 1; p < PS::COUNT; ++p) {
            const int R = PS::radix(p), ns = 1 << PS::lns(p), off = PS::twiddle_offset(p);
            for (int i = tid; i < ns * (R - 1); i += kThreads) {
                const int jm = i / (R - 1), r = i % (R - 1) + 1;
                ptw[off + i] = fft[(r * jm * (NC / ns)) / R];
            }
        }
        for (int i = tid; i < NC; i += kThreads) sp[i] = reinterpret_cast<const double2*>(P.split_tw)[i];
        for (int i = tid; i <= NC; i += kThreads) {
            const double2 r = reinterpret_cast<const double2*>(P.rot_tw)[i];
            const double h = 0.5 * sqrt(2.0 / L);
            rt[i] = r;
            rt2[i] = make_double2(r.x * h, r.y * h);
        }
        for (int i = tid; i < 4 * KT; i += kThreads) kept_idx[i] = i < P.K ? P.kept_idx[i] : -1;
        for (int i = tid; i < n_pass; i += kThreads) {
            pass_src[i] = P.pass_src[i];
            pass_dst[i] = P.pass_slot[i];
            pass_coef[i] = P.pass_coef[i];
        }
        for (int i = tid; i < 2 * TS * LDA; i += kThreads) atile[i] = 0.0;
        if (tid == 0) {
            for (int b = 0; b < 2; ++b) {
                ptx::mbar_init(&xfull[b], 1);
                ptx::mbar_init(&afull[b], kProducerThreads);
                ptx::mbar_init(&aempty[b], 32 * kConsumerWarps);
                ptx::mbar_init(&xofree[b], 1);
                ptx::mbar_init(&xempty[b], kProducerThreads);
            }
            ptx::fence_mbar_init();
        }
    }
    __syncthreads();

    const std::size_t ntiles = (batch + TS - 1) / TS;
    auto rows_of = [&](std::size_t tile) { return static_cast<int>(min(static_cast<std::size_t>(TS), batch - tile * TS)); };

    // Consumers take warpgroups 0-1 and the producer warpgroups 2-3: the warp
    // scheduler favours high warp ids, so a ready DCT instruction (2 issue
    // cycles on the shared fp64 pipe) goes ahead of a ready DMMA (16 cycles)
    // instead of starving behind the tensor work.
    constexpr int kConsumerThreads = 32 * kConsumerWarps;
    if (tid >= kConsumerThreads) {
        // =============================== producer ===================================
        // Each producer warp owns SPW = TS/8 rows of every tile and runs their
        // whole DCT warp-synchronously; the warps only meet at the mbarriers.
        asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n" ::: "memory");
        constexpr int SPW = TS / (kProducerThreads / 32);
        const int ptid = tid - kConsumerThreads, pw = ptid >> 5, lane = ptid & 31;
        // claim the next tile for buffer b and start its load (thread 0 only);
        // past the end the mbarrier is released without data
        auto claim = [&](int b) {
            const long long tile = static_cast<long long>(atomicAdd(tile_counter, 1ull));
            sched[b] = tile;
            if (tile < static_cast<long long>(ntiles)) {
                const uint32_t bytes = static_cast<uint32_t>(rows_of(tile) * n * sizeof(double));
                ptx::mbar_expect_tx(&xfull[b], bytes);
                ptx::bulk_load(xin + b * TILE, in + tile * TS * n, bytes, &xfull[b]);
            } else {
                ptx::mbar_arrive(&xfull[b]);
            }
        };
        if (ptid == 0) {
            claim(0);
            claim(1);
        }
        const double scale = sqrt(2.0 / L);
        const double dc_scale = 1.0 / sqrt(static_cast<double>(L));
        const double y_n = rt[NC].x * scale;
        bool bad = false;
        int it = 0;
        // DCTP_DEBUG_MODE & 4: per-phase cycle accounting of the producer (lane 0 of each warp)
        unsigned long long tacc[7] = {0, 0, 0, 0, 0, 0, 0};
        long long tlast = clock64();
#define T_MARK(i)                                                   \
    if (P.timers != nullptr && lane == 0) {                          \
        const long long now = clock64();                             \
        tacc[i] += static_cast<unsigned long long>(now - tlast);     \
        tlast = now;                                                 \
    }
        for (;; ++it) {
            const int b = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            T_MARK(0);
            ptx::mbar_wait(&xfull[b], ph);
            T_MARK(1);
            const long long tile = sched[b];
            if (tile >= static_cast<long long>(ntiles)) {
                // end: hand the sentinel to the consumers once they are done with buffer b
                if (it >= 2) ptx::mbar_wait(&aempty[b], ((it - 2) >> 1) & 1);
                if (ptid == 0) csched[b] = tile;
                ptx::mbar_arrive(&afull[b]);
                break;
            }
            const int valid = rows_of(tile) - pw * SPW; // rows of this warp holding real signals
            double* x = xin + b * TILE + pw * SPW * n;
            double2* xc = reinterpret_cast<double2*>(x);
            double2* cwp = cw + pw * SPW * (n / 2);
            double* ob = xout + b * TILE + pw * SPW * n;
            double* ab = atile + b * TS * LDA + pw * SPW * LDA;
            if ((P.debug & 1) == 0) {
                const double* yrow = x; // the real rows the length-L DCT reads
                if constexpr (FOLD) {
                    // the A tile of this buffer must be free before u lands in it
                    if (it >= 2) ptx::mbar_wait(&aempty[b], ((it - 2) >> 1) & 1);
                    double* ys = reinterpret_cast<double*>(cwp);
                    lane_loop<SPW * (n / 4)>(lane, [&](int t) {
                        const int r = t / (n / 4), j = 2 * (t % (n / 4));
                        const double2 lo = *reinterpret_cast<const double2*>(x + r * n + j);
                        const double2 hi = *reinterpret_cast<const double2*>(x + r * n + n - 2 - j);
                        // y_j = x_j + x_{n-1-j}, u_j = x_j - x_{n-1-j} for j, j+1
                        *reinterpret_cast<double2*>(ys + r * L + j) = make_double2(lo.x + hi.y, lo.y + hi.x);
                        *reinterpret_cast<double2*>(ab + r * LDA + j) = make_double2(lo.x - hi.y, lo.y - hi.x);
                    });
                    __syncwarp();
                    yrow = ys;
                }
                // length-L DCT-II: pass 0 reads the real rows, then ping-pong
                double2* first_dst = FOLD ? xc : cwp;
                double2* other = FOLD ? cwp : xc;
                stockham_first<NC, SPW>(yrow, first_dst, lane, valid, bad);
                __syncwarp();
                T_MARK(2);
                double2* F = fft_passes<NC, SPW, 1>(first_dst, other, ptw, lane);
                T_MARK(3);
                // real split + rotation: shat (length L) into the free buffer
                double* S = reinterpret_cast<double*>(F == cwp ? xc : cwp);
                lane_loop<SPW * (NC / 2)>(lane, [&](int t) {
                    const int r = t / (NC / 2), k = t % (NC / 2) + 1;
                    const double2* row = F + r * NC;
                    double* o = S + r * L;
                    const double2 wk = row[k], wc = row[NC - k];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int kk = h == 0 ? k : NC - k;
                        const double2 a = h == 0 ? wk : wc, c = h == 0 ? wc : wk;
                        const double sr = a.x + c.x, si = a.y - c.y; // a + conj(c)
                        const double dr = a.x - c.x, di = a.y + c.y; // a - conj(c)
                        const double2 s2 = sp[kk];
                        const double qr = s2.x * dr - s2.y * di, qi = s2.x * di + s2.y * dr;
                        const double vr = sr + qi, vi = si - qr; // 2 V_kk
                        const double2 c2 = rt2[kk];
                        o[kk] = vr * c2.x - vi * c2.y;
                        o[L - kk] = -(vr * c2.y + vi * c2.x);
                    }
                });
                if (lane < SPW) {
                    const double2 w0 = F[lane * NC];
                    const double dc = (w0.x + w0.y) * dc_scale;
                    S[lane * L] = dc;
                    S[lane * L + NC] = (w0.x - w0.y) * y_n;
                    // check_signal (fast_transform.hpp:271-276): the DC coefficient
                    // sums every sample with a nonzero weight (folded: y sums x_j and
                    // x_{n-1-j}), so an Inf/NaN input always makes it non-finite.
                    // One test per row instead of n keeps the shared fp64 pipe free.
                    if (lane < valid) bad |= !isfinite(dc);
                }
                __syncwarp();
                T_MARK(4);
                if (it >= 2) {
                    ptx::mbar_wait(&xofree[b], ((it - 2) >> 1) & 1);
                    if constexpr (!FOLD) ptx::mbar_wait(&aempty[b], ((it - 2) >> 1) & 1);
                }
                T_MARK(5);
                if constexpr (!FOLD) {
                    lane_loop<SPW * 4 * KT>(lane, [&](int t) {
                        const int r = t / (4 * KT), k = t % (4 * KT);
                        const int j = kept_idx[k];
                        if (j >= 0) ab[r * LDA + k] = S[r * L + j];
                    });
                }
                for (int q = lane; q < n_pass; q += 32) {
                    const int slotq = pass_dst[q], src = pass_src[q];
                    const double coef = pass_coef[q];
#pragma unroll
                    for (int r = 0; r < SPW; ++r) ob[r * n + slotq] = coef * S[r * L + src];
                }
                ptx::fence_proxy_async(); // pass-through writes -> visible to the consumers' TMA store
                T_MARK(6);
            } else if (it >= 2) {
                ptx::mbar_wait(&xofree[b], ((it - 2) >> 1) & 1);
                ptx::mbar_wait(&aempty[b], ((it - 2) >> 1) & 1);
            }
            __syncwarp(); // lanes finished reading S / cw before the next tile rewrites them
            if (ptid == 0) csched[b] = tile;
            ptx::mbar_arrive(&afull[b]);
            ptx::mbar_arrive(&xempty[b]); // this warp is done with xin[b] (and its cw rows)
            if (ptid == 0) {
                ptx::mbar_wait(&xempty[b], ph);
                claim(b);
            }
        }
        if (ptid == 0) release_counter(tile_counter, sched[0] + sched[1]);
        if (bad) atomicOr(flag, 1);
        if (P.timers != nullptr && lane == 0) {
            for (int i = 0; i < 7; ++i) atomicAdd(P.timers + i, tacc[i]);
            atomicAdd(P.timers + 7, static_cast<unsigned long long>(clock64() - t_entry));
            unsigned long long g_exit;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_exit));
            atomicMin(P.timers + 8, g_entry);
            atomicMax(P.timers + 9, g_exit);
            atomicMax(P.timers + 10, g_entry);
            atomicMin(P.timers + 11, g_exit);
        }
#undef T_MARK
    } else {
        // =============================== consumers ==================================
        asm volatile("setmaxnreg.inc.sync.aligned.u32 168;\n" ::: "memory");
        const int ctid = tid;
        const int warp = ctid >> 5, lane = ctid & 31;
        // Cauchy fragments, resident for the whole kernel: B[k][c] = T[k][c] for
        // this warp's NTW x 8 output columns c and all 4*KT (zero-padded) kept
        // rows, from the plan's precomputed T (row c, K contiguous).
        double bf[KT][NTW];
#pragma unroll
        for (int kt = 0; kt < KT; ++kt)
#pragma unroll
            for (int nt = 0; nt < NTW; ++nt) {
                const int k = kt * 4 + (lane & 3);
                const int c = (warp * NTW + nt) * 8 + (lane >> 2);
                bf[kt][nt] = (k < P.K && c < P.A) ? P.tmat[static_cast<std::size_t>(c) * P.K + k] : 0.0;
            }
        int slot[NTW][2];
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = (warp * NTW + nt) * 8 + 2 * (lane & 3) + e;
                slot[nt][e] = c < P.A ? P.act_slot[c] : -1;
            }
        int it = 0;
        for (;; ++it) {
            const int b = it & 1;
            ptx::mbar_wait(&afull[b], (it >> 1) & 1);
            const long long tile = csched[b];
            if (tile >= static_cast<long long>(ntiles)) break;
            const int rows = rows_of(tile);
            const double* arow = atile + b * TS * LDA + (lane >> 2) * LDA + (lane & 3);
            double acc[MT][NTW][2];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NTW; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
            for (int kt = 0; kt < KT; ++kt) {
                if (P.debug & 2) break;
                double a[MT];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) a[mt] = arow[mt * 8 * LDA + kt * 4];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                    for (int nt = 0; nt < NTW; ++nt)
                        ptx::dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], a[mt], bf[kt][nt]);
            }
            ptx::mbar_arrive(&aempty[b]);
            double* ob = xout + b * TILE;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                const int r = mt * 8 + (lane >> 2);
#pragma unroll
                for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        if (slot[nt][e] >= 0) ob[r * n + slot[nt][e]] = acc[mt][nt][e];
            }
            ptx::fence_proxy_async();
            consumer_sync();
            if (ctid == 0) {
                ptx::bulk_store(out + tile * TS * n, ob, static_cast<uint32_t>(rows * n * sizeof(double)));
                ptx::bulk_commit();
                // release the PREVIOUS tile's output buffer (its store has long
                // been read); this tile's store proceeds while we move on
                if (it >= 1) {
                    ptx::bulk_wait_read_pending1();
                    ptx::mbar_arrive(&xofree[b ^ 1]);
                }
            }
        }
        if (ctid == 0) {
            ptx::bulk_wait_all();
            if (it >= 1) ptx::mbar_arrive(&xofree[(it - 1) & 1]); // keep the phase bookkeeping exact
        }
    }
}

/// Lock-step variant: all 16 warps run the DCT phase (one row each, so the
/// fp64 pipe carries only FFT work), one CTA barrier, then the DMMA phase (one
/// 8-column N-tile each, T/W fragments resident in registers).  Tiles stream
/// through kStages TMA buffers: each buffer holds the input rows until the DCT
/// has consumed them and then collects the output rows in place; thread 0
/// issues the TMA bulk store and refills the buffer two tiles later (by then
/// the store has long finished reading it), and fetches tile indices from the
/// global counter one iteration ahead with a predicated atomic, so nothing on
/// the critical path waits for memory.  The A tile is double-buffered.  The
/// first kStages tiles of CTA b are b + q * grid (round-robin, so a small
/// batch still spreads over every CTA); later tiles come from the counter,
/// offset by kStages * grid.
constexpr int kComputeWarps = 16;
constexpr int kLockThreads = 32 * kComputeWarps;

template <bool FOLD>
constexpr int lock_stages() { return FOLD ? 4 : 3; }

template <int LOGN, int KT, int TS, bool FOLD>
constexpr std::size_t lockstep_smem_bytes() {
    constexpr int n = 1 << LOGN, L = FOLD ? n / 2 : n, NC = L / 2, TILE = TS * n;
    constexpr int tw = Passes<NC>::TWIDDLES > 0 ? Passes<NC>::TWIDDLES : 1;
    constexpr int S = lock_stages<FOLD>();
    return S * TILE * sizeof(double) + 2 * TS * NC * sizeof(double2) + 2 * TS * LDA * sizeof(double) +
           (tw + 3 * NC + 2) * sizeof(double2) + L * sizeof(double) + L * sizeof(int) +
           S * sizeof(uint64_t) + S * sizeof(long long) + 8 * sizeof(unsigned long long);
}

/// next = atomicAdd(ctr, 1) on thread 0 only, without a branch (the result is
/// consumed an iteration later, so its latency never stalls the warp).
__device__ __forceinline__ void fetch_tile_index(unsigned long long* ctr, long long& next, int tid) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.eq.u32 p, %2, 0;\n"
        "@p atom.global.add.u64 %0, [%1], 1;\n"
        "}\n"
        : "+l"(next)
        : "l"(ctr), "r"(tid)
        : "memory");
}

constexpr int kNoRoute = -(1 << 30);

template <int LOGN, int KT, int TS, bool FOLD, bool PP>
__global__ void __launch_bounds__(kLockThreads, 1)
fused_lockstep_kernel(const double* __restrict__ in, double* __restrict__ out, std::size_t batch, SmallPlanDev P,
                      int* flag, unsigned long long* tile_counter) {
    constexpr int n = 1 << LOGN, L = FOLD ? n / 2 : n, NC = L / 2, MT = TS / 8;
    constexpr int TILE = TS * n;
    constexpr int SPW = TS / kComputeWarps; // rows per warp in the DCT phase
    constexpr int kS = lock_stages<FOLD>();
    static_assert(SPW >= 1 && TS % kComputeWarps == 0, "one or more rows per warp");
    static_assert(!PP || (SPW == 1 && kS >= 4), "ping-pong: one row per warp, four stages");
    // the thread that owns the tile ring (claims, stores, scheduler counter):
    // in ping-pong mode one of the warps that start each step with the DCT
    constexpr int kDuty = PP ? 32 * (kComputeWarps / 2) : 0;
    using PS = Passes<NC>;
    extern __shared__ __align__(128) unsigned char smem[];
    double* xs = reinterpret_cast<double*>(smem);              // kS x TILE: input, then output rows
    double2* s0 = reinterpret_cast<double2*>(xs + kS * TILE);  // TS*NC complex: FFT scratch
    double2* s1 = s0 + TS * NC;                                 // TS*NC complex: FFT scratch
    double* atile = reinterpret_cast<double*>(s1 + TS * NC);   // 2 x TS x LDA: Cauchy A operand
    double2* ptw = reinterpret_cast<double2*>(atile + 2 * TS * LDA);
    double2* sp = ptw + (PS::TWIDDLES > 0 ? PS::TWIDDLES : 1);
    double2* rt = sp + NC;
    double2* rt2 = rt + NC + 1;
    // route of DCT coefficient k < L: >= 0 -> output slot (pass-through, times
    // rcoef[k]); -(c+1) -> column c of the Cauchy A tile (kept); kNoRoute -> none
    double* rcoef = reinterpret_cast<double*>(rt2 + NC + 1);
    int* route = reinterpret_cast<int*>(rcoef + L);
    uint64_t* xfull = reinterpret_cast<uint64_t*>(route + L);   // [kS] tile landed (tx bytes)
    long long* sched = reinterpret_cast<long long*>(xfull + kS);   // [kS] tile in stage q
    unsigned long long* tacc = reinterpret_cast<unsigned long long*>(sched + kS); // [8] debug phase cycles

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_pass = P.n_pass;
    {
        const double2* fft = reinterpret_cast<const double2*>(P.fft_tw);
#pragma unroll 1
        for (int p = 1; p < PS::COUNT; ++p) {
            const int R = PS::radix(p), ns = 1 << PS::lns(p), off = PS::twiddle_offset(p);
            for (int i = tid; i < ns * (R - 1); i += kLockThreads) {
                const int jm = i / (R - 1), r = i % (R - 1) + 1;
                ptw[off + i] = fft[(r * jm * (NC / ns)) / R];
            }
        }
        for (int i = tid; i < NC; i += kLockThreads) sp[i] = reinterpret_cast<const double2*>(P.split_tw)[i];
        for (int i = tid; i <= NC; i += kLockThreads) {
            const double2 r = reinterpret_cast<const double2*>(P.rot_tw)[i];
            const double h = 0.5 * sqrt(2.0 / L);
            rt[i] = r;
            rt2[i] = make_double2(r.x * h, r.y * h);
        }
        for (int i = tid; i < L; i += kLockThreads) {
            route[i] = kNoRoute;
            rcoef[i] = 0.0;
        }
        for (int i = tid; i < 2 * TS * LDA; i += kLockThreads) atile[i] = 0.0;
        __syncthreads();
        for (int i = tid; i < n_pass; i += kLockThreads) {
            route[P.pass_src[i]] = P.pass_slot[i];
            rcoef[P.pass_src[i]] = P.pass_coef[i];
        }
        if constexpr (!FOLD)
            for (int i = tid; i < P.K; i += kLockThreads) route[P.kept_idx[i]] = -(i + 1);
        if (tid == 0) {
            for (int q = 0; q < kS; ++q) ptx::mbar_init(&xfull[q], 1);
            ptx::fence_mbar_init();
        }
        if (tid < 8) tacc[tid] = 0;
    }
    // Cauchy fragments of this warp's N-tile (8 output columns), all K rows.
    double bf[KT];
    int slot[2];
    {
        const int c = warp * 8 + (lane >> 2);
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
            const int k = kt * 4 + (lane & 3);
            bf[kt] = (k < P.K && c < P.A) ? P.tmat[static_cast<std::size_t>(c) * P.K + k] : 0.0;
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int cc = warp * 8 + 2 * (lane & 3) + e;
            slot[e] = cc < P.A ? P.act_slot[cc] : -1;
        }
    }
    __syncthreads();

    const std::size_t ntiles = (batch + TS - 1) / TS;
    auto rows_of = [&](long long tile) {
        return static_cast<int>(min(static_cast<std::size_t>(TS), batch - static_cast<std::size_t>(tile) * TS));
    };
    auto claim = [&](int q, long long tile) {
        sched[q] = tile;
        if (tile < static_cast<long long>(ntiles)) {
            const uint32_t bytes = static_cast<uint32_t>(rows_of(tile) * n * sizeof(double));
            ptx::mbar_expect_tx(&xfull[q], bytes);
            ptx::bulk_load(xs + q * TILE, in + tile * TS * n, bytes, &xfull[q]);
        } else {
            ptx::mbar_arrive(&xfull[q]);
        }
    };
    long long next_tile = 0;
    if (tid == kDuty)
        for (int q = 0; q < kS; ++q) claim(q, static_cast<long long>(blockIdx.x) + q * static_cast<long long>(gridDim.x));
    fetch_tile_index(tile_counter, next_tile, tid ^ kDuty);
    const double scale = sqrt(2.0 / L);
    const double dc_scale = 1.0 / sqrt(static_cast<double>(L));
    const double y_n = rt[NC].x * scale;
    bool bad = false;
    // phase A for this warp's SPW rows of the tile in stage q: DCT (FFT, or the
    // fold's u and half-length DCT) -> Cauchy A tile `abuf`, pass-through
    // slots in place in the stage's rows
    auto dct_rows = [&](int q, long long tile, double* abuf) {
        const int valid = rows_of(tile) - warp * SPW;
        double* x = xs + q * TILE + warp * SPW * n; // this warp's rows: input, then output
        double2* a0 = s0 + warp * SPW * NC;
        double2* a1 = s1 + warp * SPW * NC;
        double* ab = abuf + warp * SPW * LDA;
        {
            const double* yrow = x;
            if constexpr (FOLD) {
                double* ys = reinterpret_cast<double*>(a1);
                lane_loop<SPW * (n / 4)>(lane, [&](int t) {
                    const int r = t / (n / 4), j = 2 * (t % (n / 4));
                    const double2 lo = *reinterpret_cast<const double2*>(x + r * n + j);
                    const double2 hi = *reinterpret_cast<const double2*>(x + r * n + n - 2 - j);
                    *reinterpret_cast<double2*>(ys + r * L + j) = make_double2(lo.x + hi.y, lo.y + hi.x);
                    *reinterpret_cast<double2*>(ab + r * LDA + j) = make_double2(lo.x - hi.y, lo.y - hi.x);
                });
                __syncwarp();
                yrow = ys;
            }
            stockham_first<NC, SPW>(yrow, a0, lane, valid, bad);
            __syncwarp();
            double2* F = fft_passes<NC, SPW, 1>(a0, a1, ptw, lane);
            // split + rotation, each coefficient routed straight to its output
            // slot (pass-through, in place: the input rows are consumed) or
            // its A-tile column (kept)
            auto emit = [&](int r, int k, double v) {
                const int rt_ = route[k];
                if (rt_ >= 0) x[r * n + rt_] = rcoef[k] * v;
                else if (rt_ != kNoRoute) ab[r * LDA + (-rt_ - 1)] = v;
            };
            lane_loop<SPW * (NC / 2)>(lane, [&](int t) {
                const int r = t / (NC / 2), k = t % (NC / 2) + 1;
                const double2* row = F + r * NC;
                const double2 wk = row[k], wc = row[NC - k];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (h == 1 && k == NC / 2) break; // self-paired
                    const int kk = h == 0 ? k : NC - k;
                    const double2 a = h == 0 ? wk : wc, c = h == 0 ? wc : wk;
                    const double sr = a.x + c.x, si = a.y - c.y;
                    const double dr = a.x - c.x, di = a.y + c.y;
                    const double2 s2 = sp[kk];
                    const double qr = s2.x * dr - s2.y * di, qi = s2.x * di + s2.y * dr;
                    const double vr = sr + qi, vi = si - qr;
                    const double2 c2 = rt2[kk];
                    emit(r, kk, vr * c2.x - vi * c2.y);
                    emit(r, L - kk, -(vr * c2.y + vi * c2.x));
                }
            });
            if (lane < SPW) {
                const double2 w0 = F[lane * NC];
                const double dc = (w0.x + w0.y) * dc_scale;
                emit(lane, 0, dc);
                emit(lane, NC, (w0.x - w0.y) * y_n);
                if (lane < valid) bad |= !isfinite(dc); // DC = sum of the row: any non-finite input shows
            }
        }
    };
    // DCTP_DEBUG_MODE & 4: phase cycles seen by thread 32 (slots 0-5) and
    // thread 0's store/claim duty (slot 6), kept in shared memory
    const bool timing = P.timers != nullptr && (tid == 32 || tid == 0);
    long long tmark = clock64();
#define LT(i)                                                        \
    if (timing) {                                                    \
        const long long now_ = clock64();                            \
        if (tid == 32 || (i) == 6) tacc[i] += static_cast<unsigned long long>(now_ - tmark); \
        tmark = now_;                                                \
    }
    if constexpr (PP) {
        // Ping-pong: step `it` multiplies tile it-1 and transforms tile it.
        // Warps 0-7 run their DMMA N-tile first and then the DCT of their row,
        // warps 8-15 the other way round, so every SMSP has one warp on the
        // fp64 tensor pipe and one on the shared-memory FFT at any time; one
        // CTA barrier per step.  The A tile is double-buffered by step parity.
        auto mma_tile = [&](int qp, const double* abuf) {
            const double* arow = abuf + (lane >> 2) * LDA + (lane & 3);
            double acc[MT][2];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
#pragma unroll
            for (int kt = 0; kt < KT; ++kt) {
                double a[MT];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) a[mt] = arow[mt * 8 * LDA + kt * 4];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) ptx::dmma_8x8x4(acc[mt][0], acc[mt][1], a[mt], bf[kt]);
            }
            double* obt = xs + qp * TILE;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                const int r = mt * 8 + (lane >> 2);
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    if (slot[e] >= 0) obt[r * n + slot[e]] = acc[mt][e];
            }
        };
        ptx::mbar_wait(&xfull[0], 0);
        dct_rows(0, sched[0], atile); // grid <= tiles: every CTA owns tile sched[0]
        __syncthreads();
        for (int it = 1;; ++it) {
            const int q = it % kS, qp = (it - 1) % kS;
            const long long tprev = sched[qp];
            bool live = false;
            auto dct_step = [&] {
                ptx::mbar_wait(&xfull[q], (it / kS) & 1);
                const long long tile = sched[q];
                live = tile < static_cast<long long>(ntiles);
                if (live) dct_rows(q, tile, atile + (it & 1) * TS * LDA);
            };
            // DCTP_DEBUG_MODE & 4: lane 0 of warps 0 / 8 time part 1, part 2 and the
            // barrier wait (timer slots 0-2 / 3-5)
            const bool ptime = P.timers != nullptr && (tid == 0 || tid == kDuty);
            const long long t0 = ptime ? clock64() : 0;
            long long t1 = 0;
            if (warp < kComputeWarps / 2) {
                mma_tile(qp, atile + ((it - 1) & 1) * TS * LDA);
                if (ptime) t1 = clock64();
                dct_step();
            } else {
                dct_step();
                if (ptime) t1 = clock64();
                mma_tile(qp, atile + ((it - 1) & 1) * TS * LDA);
            }
            const long long t2 = ptime ? clock64() : 0;
            ptx::fence_proxy_async(); // output writes -> the TMA store below
            __syncthreads();
            if (ptime) {
                const int b = tid == 0 ? 0 : 3;
                atomicAdd(P.timers + b, static_cast<unsigned long long>(t1 - t0));
                atomicAdd(P.timers + b + 1, static_cast<unsigned long long>(t2 - t1));
                atomicAdd(P.timers + b + 2, static_cast<unsigned long long>(clock64() - t2));
            }
            if (tid == kDuty) {
                ptx::bulk_store(out + tprev * TS * n, xs + qp * TILE,
                                static_cast<uint32_t>(rows_of(tprev) * n * sizeof(double)));
                ptx::bulk_commit();
                if (it >= 2) {
                    // refill the stage of tile it-2: its store (issued a step ago) has been read
                    ptx::bulk_wait_read_pending1();
                    claim((it - 2) % kS, next_tile + kS * static_cast<long long>(gridDim.x));
                }
            }
            if (it >= 2) fetch_tile_index(tile_counter, next_tile, tid ^ kDuty);
            if (!live) break;
        }
    } else {
    for (int it = 0;; ++it) {
        const int q = it % kS;
        LT(5);
        ptx::mbar_wait(&xfull[q], (it / kS) & 1);
        LT(0);
        const long long tile = sched[q];
        if (tile >= static_cast<long long>(ntiles)) break;
        double* abuf = atile + (it & 1) * TS * LDA;
        // ---- phase A: DCT of this warp's rows --------------------------------------
        if ((P.debug & 1) == 0) dct_rows(q, tile, abuf);
        LT(1);
        __syncthreads(); // A tile (and in-place pass-through rows) complete
        LT(2);
        // ---- phase B: DMMA, this warp's 8 columns for all TS rows ----------------
        {
            const double* arow = abuf + (lane >> 2) * LDA + (lane & 3);
            double acc[MT][2];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
#pragma unroll
            for (int kt = 0; kt < KT; ++kt) {
                if (P.debug & 2) break;
                double a[MT];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) a[mt] = arow[mt * 8 * LDA + kt * 4];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) ptx::dmma_8x8x4(acc[mt][0], acc[mt][1], a[mt], bf[kt]);
            }
            double* obt = xs + q * TILE;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                const int r = mt * 8 + (lane >> 2);
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    if (slot[e] >= 0) obt[r * n + slot[e]] = acc[mt][e];
            }
        }
        LT(3);
        ptx::fence_proxy_async(); // output writes -> the TMA store below
        __syncthreads();
        LT(4);
        if (tid == kDuty) {
            ptx::bulk_store(out + tile * TS * n, xs + q * TILE, static_cast<uint32_t>(rows_of(tile) * n * sizeof(double)));
            ptx::bulk_commit();
            if (it >= 1) {
                // refill the stage of tile it-1: its store is (all but) certainly read
                ptx::bulk_wait_read_pending1();
                claim((it - 1) % kS, next_tile + kS * static_cast<long long>(gridDim.x));
            }
        }
        LT(6);
        if (it >= 1) fetch_tile_index(tile_counter, next_tile, tid ^ kDuty); // used next iteration
    }
    }
#undef LT
    if (timing) {
        if (tid == 32)
            for (int i = 0; i < 6; ++i) atomicAdd(P.timers + i, tacc[i]);
        if (tid == 0) atomicAdd(P.timers + 6, tacc[6]);
    }
    if (bad) atomicOr(flag, 1);
    if (tid == kDuty) {
        ptx::bulk_wait_all();
        release_counter(tile_counter, next_tile);
    }
}

template <int LOGN, int KT, int TS, bool FOLD>
constexpr std::size_t smem_bytes() {
    constexpr int n = 1 << LOGN, L = FOLD ? n / 2 : n, NC = L / 2, TILE = TS * n;
    constexpr int tw = Passes<NC>::TWIDDLES > 0 ? Passes<NC>::TWIDDLES : 1;
    return 4 * TILE * sizeof(double) + (TILE / 2) * sizeof(double2) + 2 * TS * LDA * sizeof(double) +
           (tw + 3 * NC + 2) * sizeof(double2) + n * sizeof(double) + (4 * KT + 2 * n) * sizeof(int) +
           10 * sizeof(uint64_t) + 4 * sizeof(long long);
}

/// Scheduler counter pair of (current device, stream), allocated and zeroed
/// once; the kernels leave it zeroed (release_counter).  Keyed by
/// cudaStreamGetId, not the handle: cudaStreamPerThread (or the null stream
/// under per-thread default streams) is one handle for many real streams, and
/// a destroyed stream's handle can be reused while its kernels still run.
cudaError_t stream_counter(cudaStream_t stream, unsigned long long** out) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<int, unsigned long long>, unsigned long long*>> reg;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    unsigned long long sid = 0;
    e = cudaStreamGetId(stream, &sid);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    for (auto& r : reg)
        if (r.first.first == dev && r.first.second == sid) {
            *out = r.second;
            return cudaSuccess;
        }
    unsigned long long* c = nullptr;
    e = cudaMalloc(reinterpret_cast<void**>(&c), 2 * sizeof(unsigned long long));
    if (e != cudaSuccess) return e;
    e = cudaMemset(c, 0, 2 * sizeof(unsigned long long));
    if (e != cudaSuccess) return e;
    reg.push_back({{dev, sid}, c});
    *out = c;
    return cudaSuccess;
}

template <int LOGN, int NTW, int KT, bool FOLD>
cudaError_t launch_small(const double* in, double* out, std::size_t batch, const SmallPlanDev& P, int* flag,
                         int num_sms, cudaStream_t stream) {
    constexpr int TS = LOGN >= 9 ? 8 : 16;
    std::size_t smem = smem_bytes<LOGN, KT, TS, FOLD>();
    static_assert(smem_bytes<LOGN, KT, TS, FOLD>() <= 227 * 1024, "fused small kernel exceeds shared memory");
    static const bool lockstep = [] {
        const char* e = std::getenv("DCTP_FUSED_VARIANT");
        return !(e && std::string(e) == "specialised");
    }();
    auto kern = fused_small_fwd_kernel<LOGN, NTW, KT, TS, FOLD>;
    int threads = kThreads;
    if constexpr (TS >= kComputeWarps) {
        static_assert(lockstep_smem_bytes<LOGN, KT, TS, FOLD>() <= 227 * 1024, "lockstep kernel exceeds shared memory");
        if (lockstep && NTW == 1) {
            kern = fused_lockstep_kernel<LOGN, KT, TS, FOLD, false>;
            if constexpr (FOLD && TS / kComputeWarps == 1 && lock_stages<FOLD>() >= 4) {
                static const bool pp = [] {
                    const char* e = std::getenv("DCTP_FUSED_VARIANT");
                    return !(e && std::string(e) == "lockstep");
                }();
                if (pp) kern = fused_lockstep_kernel<LOGN, KT, TS, FOLD, true>;
            }
            smem = lockstep_smem_bytes<LOGN, KT, TS, FOLD>();
            threads = kLockThreads;
        }
    }
    const cudaError_t attr = smem_optin(reinterpret_cast<const void*>(kern), static_cast<int>(smem));
    if (attr != cudaSuccess) return attr;
    const std::size_t ntiles = (batch + TS - 1) / TS;
    const unsigned grid = static_cast<unsigned>(std::min<std::size_t>(ntiles, static_cast<std::size_t>(num_sms)));
    // tile counter: one self-re-arming pair per (device, stream) — launches on
    // one stream are ordered, launches on different streams get different
    // pairs; under stream capture a fresh pair from the stream-ordered pool
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(stream, &cap);
    if (e != cudaSuccess) return e;
    if (cap != cudaStreamCaptureStatusNone) {
        unsigned long long* counter = nullptr;
        e = cudaMallocAsync(reinterpret_cast<void**>(&counter), 2 * sizeof(unsigned long long), stream);
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(counter, 0, 2 * sizeof(unsigned long long), stream);
        if (e != cudaSuccess) return e;
        kern<<<grid, threads, smem, stream>>>(in, out, batch, P, flag, counter);
        e = cudaGetLastError();
        cudaFreeAsync(counter, stream);
        return e;
    }
    unsigned long long* counter = nullptr;
    e = stream_counter(stream, &counter);
    if (e != cudaSuccess) return e;
    kern<<<grid, threads, smem, stream>>>(in, out, batch, P, flag, counter);
    return cudaGetLastError();
}

template <int LOGN, int KT, bool FOLD>
cudaError_t dispatch_ntw(const double* in, double* out, std::size_t batch, const SmallPlanDev& P, int* flag,
                         int num_sms, cudaStream_t stream) {
    static const bool specialised = [] {
        const char* e = std::getenv("DCTP_FUSED_VARIANT");
        return e && std::string(e) == "specialised";
    }();
    if (!specialised || P.A <= 8 * kConsumerWarps)
        return launch_small<LOGN, 1, KT, FOLD>(in, out, batch, P, flag, num_sms, stream);
    return launch_small<LOGN, 2, KT, FOLD>(in, out, batch, P, flag, num_sms, stream);
}

/// K is padded up to 4*KT with KT in {4, 8, 16, 32} (never above n/4).  A
/// folded plan's Cauchy K is n/2.
template <int LOGN>
cudaError_t dispatch_kt(const double* in, double* out, std::size_t batch, const SmallPlanDev& P, int* flag,
                        int num_sms, cudaStream_t stream) {
    constexpr int n = 1 << LOGN;
    if constexpr (n >= 64 && n / 8 <= KTMAX) {
        if (P.fold) return dispatch_ntw<LOGN, n / 8, true>(in, out, batch, P, flag, num_sms, stream);
    }
    if (P.fold) return cudaErrorInvalidValue;
    if (P.K <= 16 || n <= 16) return dispatch_ntw<LOGN, 4, false>(in, out, batch, P, flag, num_sms, stream);
    if constexpr (n >= 32)
        if (P.K <= 32 || n <= 32) return dispatch_ntw<LOGN, 8, false>(in, out, batch, P, flag, num_sms, stream);
    if constexpr (n >= 64)
        if (P.K <= 64 || n <= 64) return dispatch_ntw<LOGN, 16, false>(in, out, batch, P, flag, num_sms, stream);
    if constexpr (n >= 128) return dispatch_ntw<LOGN, 32, false>(in, out, batch, P, flag, num_sms, stream);
    return cudaErrorInvalidValue;
}

} // namespace

bool fused_small_supported(std::size_t n, int K, int A) {
    return is_pow2(n) && n >= 16 && n <= 512 && K <= 4 * KTMAX && A <= 16 * kConsumerWarps;
}

bool fused_small_fold_supported(std::size_t n, int columns) {
    return is_pow2(n) && n >= 64 && n / 2 <= 4 * KTMAX && columns <= 16 * kConsumerWarps;
}

cudaError_t fused_small_forward(const double* in, double* out, std::size_t batch, const SmallPlanDev& P, int* flag,
                                int num_sms, cudaStream_t stream) {
    if (batch == 0) return cudaSuccess;
    switch (P.n) {
        case 16: return dispatch_kt<4>(in, out, batch, P, flag, num_sms, stream);
        case 32: return dispatch_kt<5>(in, out, batch, P, flag, num_sms, stream);
        case 64: return dispatch_kt<6>(in, out, batch, P, flag, num_sms, stream);
        case 128: return dispatch_kt<7>(in, out, batch, P, flag, num_sms, stream);
        case 256: return dispatch_kt<8>(in, out, batch, P, flag, num_sms, stream);
        case 512: return dispatch_kt<9>(in, out, batch, P, flag, num_sms, stream);
        default: return cudaErrorInvalidValue;
    }
}

} // namespace dctp::dev
