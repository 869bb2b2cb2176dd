// The reference's fast route on the GPU (fp64): DCT-II, DST-I, a
// nonuniform fast sine transform (NFST) by Gaussian gridding, and the
// secular-row epilogue, for one signal per CTA entirely in shared memory.
//
// Reference: DctPlusPlan::forward (proj/include/dctplus/fast_transform.hpp:
// 163-190) with NfstPlan::exec_into (nfst.hpp:201-238).  Per signal:
//   shat = DCT-II(s); sv = z .* shat; out[pass] = sigma shat[src];
//   out[ext] = scale_ext * <ext_row, sv>;
//   h_j = w_j sv_j,  w_j = (-1)^(j+1) / sin(j pi / n)          (j = 1..n-1)
//   c = DST-I(h);  v_k = c_k / phi_hat(k)                      (deconvolution)
//   y_l = Im g_l = 2 sum_k v_k sin(pi k l / 2n)                (grid G = 4n)
//   phi_r = 1/2 sum_t w_rt y_{lo_r + t}                        (35 taps)
//   out[slot_r] = scale_r (-phi_r / (2 sin(n theta_r)) + sv_0 / nu_r).
// The grid transform is split by the parity of l: y_{2k} = DST-I(v)_k and
// y_{2k+1} = (-1)^k DCT-III(v reversed)_k, so every FFT has length <= n and
// the row fits in shared memory up to n = 8192 (in-place FFTs, 209 KB).
// The Gaussian weights are w_rt = P0_r B_r^t C_t (fast Gaussian gridding):
// two per-target constants and one shared 35-entry table instead of the
// reference's 35 weights per target.
#include <algorithm>

#include "kernels/common.cuh"
#include "kernels/fft_smem.cuh"
#include "kernels/launch.hpp"

namespace dctp::dev {
namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

/// Block-wide sum; `red` holds >= 33 doubles.  Every thread gets the total.
__device__ __forceinline__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double t = lane < static_cast<int>(blockDim.x >> 5) ? red[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) red[32] = t;
    }
    __syncthreads();
    return red[32];
}

/// The odd extension e (length 2n) of h_1..h_{n-1} packed as z_j = e_{2j} +
/// i e_{2j+1} (j < n): its n-point FFT gives DST-I(h) in dst1_pair below.
__device__ __forceinline__ double odd_ext(const double* h, const double* wgt, int i, int n) {
    if (i == 0 || i == n) return 0.0;
    if (i < n) return wgt ? wgt[i] * h[i] : h[i];
    const int k = 2 * n - i;
    return -(wgt ? wgt[k] * h[k] : h[k]);
}

/// (stored at the bit-reversed positions the FFT's first pass reads)
__device__ __forceinline__ void pack_dst1(double2* cb, const double* h, const double* __restrict__ wgt, int n,
                                          int logn) {
    for (int j = threadIdx.x; j < n; j += blockDim.x)
        cb[pad8(static_cast<int>(bit_reverse(static_cast<unsigned>(j), logn)))] =
            make_double2(odd_ext(h, wgt, 2 * j, n), odd_ext(h, wgt, 2 * j + 1, n));
}

__device__ __forceinline__ int brev(int i, int bits) {
    return static_cast<int>(bit_reverse(static_cast<unsigned>(i), bits));
}

/// c_k and c_{n-k} of DST-I (c_k = 2 sum_j h_j sin(pi j k / n)) from the
/// n-point FFT Z of the packed odd extension: E_k = Ev_k + W^k Od_k with
/// Ev = (Z_k + conj Z_{n-k}) / 2, Od = (Z_k - conj Z_{n-k}) / 2i, W = e^{-i pi/n},
/// and E_k = -i c_k.
__device__ __forceinline__ void dst1_pair(double2 a, double2 b, double2 w, double& ck, double& cnk) {
    // k: A = Z_k, B = Z_{n-k}
    const double ev_y = 0.5 * (a.y - b.y);
    const double od_x = 0.5 * (a.y + b.y), od_y = -0.5 * (a.x - b.x);
    ck = -(ev_y + w.x * od_y + w.y * od_x);
    // n-k: roles swapped, W^{n-k} = (-w.x, w.y)
    const double ev2_y = 0.5 * (b.y - a.y);
    const double od2_x = 0.5 * (b.y + a.y), od2_y = -0.5 * (b.x - a.x);
    cnk = -(ev2_y - w.x * od2_y + w.y * od2_x);
}

/// DST-I of the packed row in cb (after its FFT) into dst[1..n-1] (dst[0] = 0),
/// optionally multiplied by mul[k].
__device__ __forceinline__ void unpack_dst1(const double2* cb, const double* __restrict__ tw2n,
                                            const double* __restrict__ mul, double* dst, int n) {
    const int N = n >> 1;
    for (int k = threadIdx.x; k <= N; k += blockDim.x) {
        if (k == 0) {
            dst[0] = 0.0;
            continue;
        }
        const double2 w = __ldg(reinterpret_cast<const double2*>(tw2n) + k);
        double ck, cnk;
        dst1_pair(cb[pad8(k)], cb[pad8(n - k)], w, ck, cnk);
        dst[k] = mul ? ck * __ldg(mul + k) : ck;
        if (k != N) dst[n - k] = mul ? cnk * __ldg(mul + n - k) : cnk;
    }
}

/// Halo of the grid arrays: the tap windows of targets near theta = 0 / pi
/// reach past l = 0 / 2n, where y is odd-reflected (y_{-l} = -y_l, y_{2n+l} =
/// -y_{2n-l}); the arrays carry the reflected values so the tap loops run
/// branch-free.  kHalo >= (halfwidth + 3) / 2 for halfwidth <= 28.
constexpr int kHalo = 16;

/// Complex entries of the FFT row: the n-point FFT, or the n/2-point FFT
/// plus the odd-grid array (n reals + halos) beside it.
__host__ __device__ constexpr int cb_len(int n) {
    return padded_len(n) > padded_len(n / 2) + (n + 2 * kHalo) / 2 + 1 ? padded_len(n)
                                                                       : padded_len(n / 2) + (n + 2 * kHalo) / 2 + 1;
}

/// Sum (or, SPREAD, scatter-add of phi times) the taps of one parity of one
/// target: l = lo + t, t = 0..2 hw, parity ODD, on the array y indexed by
/// floor(l / 2) (halos included).  Weights w_t = P0 B^t C_t by the
/// recurrence w_{t+2} = w_t G, G_{t+2} = G_t E with G_t = B^2 C_{t+2} / C_t
/// (Gaussian: C_{t+2} / C_t = exp(-4 alpha (t - hw + 1)), E = exp(-8 alpha));
/// g = {C_0, C_1, R_0, R_1, E}, R_t0 = C_{t0+2} / C_t0.
template <int HW, bool ODD, bool SPREAD>
__device__ __forceinline__ double tap_pass(double* y, int lo, double p0, double B, const double* g, int hw_rt,
                                           double phi = 0.0) {
    const int hw = HW > 0 ? HW : hw_rt;
    const int t0 = (((lo & 1) != 0) == ODD) ? 0 : 1;
    double* yy = y + ((lo + t0 - (ODD ? 1 : 0)) >> 1);
    double w = p0 * (t0 ? B * g[1] : g[0]);
    if (SPREAD) w *= phi;
    double G = B * B * (t0 ? g[3] : g[2]);
    const double E = g[4];
    const int K = hw + 1 - t0;
    double a = 0.0;
    if constexpr (HW > 0) {
#pragma unroll
        for (int k = 0; k <= HW; ++k) {
            if (k < K) {
                if (SPREAD)
                    atomicAdd(yy + k, w);
                else
                    a = fma(w, yy[k], a);
            }
            w *= G;
            G *= E;
        }
    } else {
        for (int k = 0; k < K; ++k) {
            if (SPREAD)
                atomicAdd(yy + k, w);
            else
                a = fma(w, yy[k], a);
            w *= G;
            G *= E;
        }
    }
    return a;
}

template <bool ODD, bool SPREAD>
__device__ __forceinline__ double taps(const FastPlanDev& P, double* y, int r, const double* g, double phi = 0.0) {
    const int lo = __ldg(P.t_lo + r);
    const double p0 = __ldg(P.t_p0 + r), B = __ldg(P.t_b + r);
    if (P.hw == 17) return tap_pass<17, ODD, SPREAD>(y, lo, p0, B, g, 17, phi);
    return tap_pass<0, ODD, SPREAD>(y, lo, p0, B, g, P.hw, phi);
}

/// Odd-reflected halos: yo[i] = y_{2i+1} and ye[i] = y_{2i} (ye[0] = ye[n] = 0).
__device__ __forceinline__ void fill_halos(double* yo, double* ye, int n) {
    for (int k = threadIdx.x; k < kHalo; k += blockDim.x) {
        if (yo) {
            yo[-k - 1] = -yo[k];
            yo[n + k] = -yo[n - 1 - k];
        }
        if (ye) {
            if (k == 0) {
                ye[n] = 0.0;
            } else {
                ye[-k] = -ye[k];
                ye[n + k] = -ye[n - k];
            }
        }
    }
}

__global__ void __launch_bounds__(512)
nfst_forward_kernel(const double* __restrict__ in, double* __restrict__ out, FastPlanDev P, int* flag) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = P.n, logn = P.logn, N = n >> 1;
    double2* cb = reinterpret_cast<double2*>(smem_raw);                // FFT row, cb_len(n) complex
    double* rb = reinterpret_cast<double*>(cb + cb_len(n)) + kHalo;    // n reals: shat, then v, then y_even
    double* g = rb + n + kHalo;                                         // 5 weight-recurrence constants
    double* red = g + 8;                                                // 33
    double* yo = reinterpret_cast<double*>(cb + padded_len(N)) + kHalo; // y_odd, beside the n/2-point FFT
    const std::size_t b = blockIdx.x;
    const double* x = in + b * n;
    double* o = out + b * n;
    const int tid = threadIdx.x, nt = blockDim.x;

    if (tid < 5) g[tid] = __ldg(P.ctab + tid);

    // 1. DCT-II (Makhoul): v = (x0, x2, ..., x3, x1) packed as w_m = v_2m + i v_2m+1
    bool bad = false;
    for (int j = tid; j < n; j += nt) {
        const double v = x[j];
        bad |= !isfinite(v);
        const int p = (j & 1) ? (n - 1 - (j >> 1)) : (j >> 1);
        reinterpret_cast<double*>(&cb[pad8(brev(p >> 1, logn - 1))])[p & 1] = v;
    }
    if (bad) atomicOr(flag, 1);
    __syncthreads();
    fft_from_bitreversed<double, false>(cb, N, logn - 1, P.tw2n, 2);
    {
        const double scale = sqrt(2.0 / n), dc_scale = 1.0 / sqrt(static_cast<double>(n));
        const double2* tw = reinterpret_cast<const double2*>(P.tw2n);
        const double2* rot = reinterpret_cast<const double2*>(P.rot);
        for (int k = tid; k < N; k += nt) {
            if (k == 0) {
                const double2 w0 = cb[0];
                rb[0] = (w0.x + w0.y) * dc_scale;
                rb[N] = (w0.x - w0.y) * __ldg(&rot[N].x) * scale;
                continue;
            }
            const double2 wk = cb[pad8(k)], wc = cb[pad8(N - k)];
            const double er = 0.5 * (wk.x + wc.x), ei = 0.5 * (wk.y - wc.y);
            const double orr = 0.5 * (wk.x - wc.x), oi = 0.5 * (wk.y + wc.y);
            const double2 sp = __ldg(tw + 2 * k); // e^{-2 pi i k / n}
            const double qr = sp.x * orr - sp.y * oi, qi = sp.x * oi + sp.y * orr;
            const double vr = er + qi, vi = ei - qr;
            const double2 rt = __ldg(rot + k);
            rb[k] = (vr * rt.x - vi * rt.y) * scale;
            rb[n - k] = -(vr * rt.y + vi * rt.x) * scale;
        }
    }
    __syncthreads();

    // 2. pass-through slots, the exterior row, sv_0; h = w .* z .* shat packed for DST-I
    for (int e = tid; e < P.n_pass; e += nt) o[__ldg(P.pass_slot + e)] = __ldg(P.pass_sign + e) * rb[__ldg(P.pass_src + e)];
    const double sv0 = P.z0 * rb[0];
    double ext = 0.0;
    if (P.ext_slot >= 0)
        for (int j = tid; j < n; j += nt) ext += __ldg(P.ez + j) * rb[j];
    pack_dst1(cb, rb, P.hz, n, logn);
    if (P.ext_slot >= 0) {
        ext = block_sum(ext, red); // includes the barrier before the FFT
        if (tid == 0) o[P.ext_slot] = P.ext_scale * ext;
    } else {
        __syncthreads();
    }

    // 3. c = DST-I(h); v = c / phi_hat
    fft_from_bitreversed<double, false>(cb, n, logn, P.tw2n, 1);
    unpack_dst1(cb, P.tw2n, P.inv_phi, rb, n);
    __syncthreads();

    // 4. odd grid points: y_{2k+1} = (-1)^k core DCT-III of X, X_0 = 0, X_m = 2 v_{n-m}
    {
        const double2* tw = reinterpret_cast<const double2*>(P.tw2n);
        const double2* rot = reinterpret_cast<const double2*>(P.rot);
        const double r2 = 0.70710678118654752440;
        for (int k = tid; k < N; k += nt) {
            const double2 rt = __ldg(rot + k);
            const double cr = rt.x, ci = -rt.y; // e^{+i pi k / 2n}
            const double ar = (k == 0) ? 0.0 : 2.0 * rb[n - k];
            const double ai = (k == 0) ? 0.0 : -2.0 * rb[k];
            const double v1r = ar * cr - ai * ci, v1i = ar * ci + ai * cr;
            const double c2r = r2 * (cr - ci), c2i = r2 * (cr + ci);
            const double br = 2.0 * rb[N - k], bi = -2.0 * rb[N + k];
            const double v2r = br * c2r - bi * c2i, v2i = br * c2i + bi * c2r;
            const double2 sp = __ldg(tw + 2 * k);
            const double sr = sp.x, si = -sp.y; // e^{+2 pi i k / n}
            const double dr = v1r - v2r, di = v1i - v2i;
            const double qr = sr * dr - si * di, qi = sr * di + si * dr;
            cb[pad8(brev(k, logn - 1))] = make_double2(0.5 * (v1r + v2r - qi), 0.5 * (v1i + v2i + qr));
        }
    }
    __syncthreads();
    fft_from_bitreversed<double, true>(cb, N, logn - 1, P.tw2n, 2);
    for (int j = tid; j < n; j += nt) {
        const int p = (j & 1) ? (n - 1 - (j >> 1)) : (j >> 1);
        const double2 w = cb[pad8(p >> 1)];
        const double v = (p & 1) ? w.y : w.x;
        yo[j] = (j & 1) ? -v : v;
    }
    __syncthreads();

    fill_halos(yo, nullptr, n);
    __syncthreads();

    // 5. gather the odd taps of every interior target; the partial sum parks
    //    in the target's own output slot (same thread reads it back in 7)
    for (int r = tid; r < P.R; r += nt) o[__ldg(P.t_slot + r)] = taps<true, false>(P, yo, r, g);
    __syncthreads();

    // 6. even grid points: y_{2k} = DST-I(v)_k
    pack_dst1(cb, rb, nullptr, n, logn);
    __syncthreads();
    fft_from_bitreversed<double, false>(cb, n, logn, P.tw2n, 1);
    unpack_dst1(cb, P.tw2n, nullptr, rb, n);
    __syncthreads();

    fill_halos(nullptr, rb, n);
    __syncthreads();

    // 7. even taps, then the secular-row epilogue
    for (int r = tid; r < P.R; r += nt) {
        const int slot = __ldg(P.t_slot + r);
        const double a = o[slot] + taps<false, false>(P, rb, r, g);
        o[slot] = __ldg(P.t_ca + r) * a + __ldg(P.t_cb + r) * sv0;
    }
}

/// Inverse through the adjoint NFST (DctPlusPlan::inverse(p, ws, fast = true),
/// fast_transform.hpp:218-255 with NfstPlan::adjoint_into, nfst.hpp:248-277):
///   phi_r = -y_r / (2 sin(n theta_r)), y_r = -scale_r p[slot_r];
///   f = spread of phi over the grid; b_k = Im(FFT f)_k / phi_hat(k), split
///   by parity as 1/2 DST-I(f_even)_k + DCT-II(+-f_odd)_{n-k};
///   g = DST-I(b); d_j = z_j (ext_j + [j = 0] d0 - w_j g_j) + pass-through;
///   s = DCT-III(d).
__global__ void __launch_bounds__(512)
nfst_inverse_kernel(const double* __restrict__ in, double* __restrict__ out, FastPlanDev P, int* flag) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = P.n, logn = P.logn, N = n >> 1;
    double2* cb = reinterpret_cast<double2*>(smem_raw);
    double* rb = reinterpret_cast<double*>(cb + cb_len(n)) + kHalo;
    double* g = rb + n + kHalo;
    double* red = g + 8;
    double* fo = reinterpret_cast<double*>(cb + padded_len(N)) + kHalo; // odd grid points, beside the n/2-point FFT
    const std::size_t b = blockIdx.x;
    const double* prow = in + b * n;
    double* o = out + b * n;
    const int tid = threadIdx.x, nt = blockDim.x;
    const double2* tw = reinterpret_cast<const double2*>(P.tw2n);
    const double2* rot = reinterpret_cast<const double2*>(P.rot);

    if (tid < 5) g[tid] = __ldg(P.ctab + tid);
    bool bad = false;
    for (int j = tid; j < n; j += nt) bad |= !isfinite(prow[j]);
    for (int j = tid - kHalo; j < n + kHalo; j += nt) rb[j] = 0.0;
    if (bad) atomicOr(flag, 1);
    __syncthreads();

    // 1. even grid points -> c = DST-I(f_even) (kept in rb); the halos fold
    //    back with the odd reflection (the adjoint of fill_halos)
    for (int r = tid; r < P.R; r += nt) taps<false, true>(P, rb, r, g, -2.0 * __ldg(P.t_ca + r) * prow[__ldg(P.t_slot + r)]);
    __syncthreads();
    for (int k = tid + 1; k < kHalo; k += nt) {
        rb[k] -= rb[-k];
        rb[n - k] -= rb[n + k];
    }
    __syncthreads();
    pack_dst1(cb, rb, nullptr, n, logn);
    __syncthreads();
    fft_from_bitreversed<double, false>(cb, n, logn, P.tw2n, 1);
    unpack_dst1(cb, P.tw2n, nullptr, rb, n);
    __syncthreads();

    // 2. odd grid points -> Y = DCT-II core of (-1)^j f_odd_j (Makhoul, n/2 points)
    for (int j = tid - kHalo; j < n + kHalo; j += nt) fo[j] = 0.0;
    __syncthreads();
    for (int r = tid; r < P.R; r += nt) taps<true, true>(P, fo, r, g, -2.0 * __ldg(P.t_ca + r) * prow[__ldg(P.t_slot + r)]);
    __syncthreads();
    for (int k = tid; k < kHalo; k += nt) {
        fo[k] -= fo[-k - 1];
        fo[n - 1 - k] -= fo[n + k];
    }
    __syncthreads();
    for (int j = tid; j < n; j += nt) {
        const double v = (j & 1) ? -fo[j] : fo[j];
        const int q = (j & 1) ? (n - 1 - (j >> 1)) : (j >> 1);
        // the n/2-point FFT row (cb head) and fo (cb tail) are disjoint
        reinterpret_cast<double*>(&cb[pad8(brev(q >> 1, logn - 1))])[q & 1] = v;
    }
    __syncthreads();
    fft_from_bitreversed<double, false>(cb, N, logn - 1, P.tw2n, 2);
    // b_k = inv_phi_k (c_k / 2 + Y_{n-k}); Y_q for q = 1..n-1 from the split
    for (int k = tid; k < N; k += nt) {
        double yk, ynk; // Y_k, Y_{n-k}
        if (k == 0) {
            const double2 w0 = cb[0];
            yk = 0.0; // Y_0 is not used (b_n does not exist)
            ynk = (w0.x - w0.y) * __ldg(&rot[N].x); // Y_N
            rb[N] = __ldg(P.inv_phi + N) * (0.5 * rb[N] + ynk);
            continue;
        }
        const double2 wk = cb[pad8(k)], wc = cb[pad8(N - k)];
        const double er = 0.5 * (wk.x + wc.x), ei = 0.5 * (wk.y - wc.y);
        const double orr = 0.5 * (wk.x - wc.x), oi = 0.5 * (wk.y + wc.y);
        const double2 sp = __ldg(tw + 2 * k);
        const double qr = sp.x * orr - sp.y * oi, qi = sp.x * oi + sp.y * orr;
        const double vr = er + qi, vi = ei - qr;
        const double2 rt = __ldg(rot + k);
        yk = vr * rt.x - vi * rt.y;
        ynk = -(vr * rt.y + vi * rt.x);
        // b_{n-k} uses Y_k, b_k uses Y_{n-k}
        rb[k] = __ldg(P.inv_phi + k) * (0.5 * rb[k] + ynk);
        rb[n - k] = __ldg(P.inv_phi + n - k) * (0.5 * rb[n - k] + yk);
    }
    __syncthreads();

    // 3. g = DST-I(b); d = z (ext + d0 e_0 - w g) + pass-through, into rb
    pack_dst1(cb, rb, nullptr, n, logn);
    double d0 = 0.0;
    for (int r = tid; r < P.R; r += nt) d0 += __ldg(P.t_cb + r) * prow[__ldg(P.t_slot + r)];
    d0 = block_sum(d0, red); // barrier: the pack is complete
    const double pe = P.ext_slot >= 0 ? P.ext_scale * prow[P.ext_slot] : 0.0;
    fft_from_bitreversed<double, false>(cb, n, logn, P.tw2n, 1);
    for (int k = tid; k <= N; k += nt) {
        double gk, gnk;
        if (k == 0) {
            rb[0] = P.z0 * d0 + (P.ext_slot >= 0 ? pe * __ldg(P.ez) : 0.0);
            continue;
        }
        dst1_pair(cb[pad8(k)], cb[pad8(n - k)], __ldg(tw + k), gk, gnk);
        const double ek = P.ext_slot >= 0 ? pe * __ldg(P.ez + k) : 0.0;
        rb[k] = ek - __ldg(P.hz + k) * gk;
        if (k != N) {
            const double enk = P.ext_slot >= 0 ? pe * __ldg(P.ez + n - k) : 0.0;
            rb[n - k] = enk - __ldg(P.hz + n - k) * gnk;
        }
    }
    __syncthreads();
    for (int e = tid; e < P.n_pass; e += nt)
        rb[__ldg(P.pass_src + e)] += __ldg(P.pass_sign + e) * prow[__ldg(P.pass_slot + e)];
    __syncthreads();

    // 4. s = orthonormal DCT-III(d) (Makhoul, n/2 points)
    {
        const double scale = sqrt(2.0 / n), dc = 2.0 / sqrt(static_cast<double>(n));
        const double r2 = 0.70710678118654752440;
        for (int k = tid; k < N; k += nt) {
            const double2 rt = __ldg(rot + k);
            const double cr = rt.x, ci = -rt.y;
            const double ar = (k == 0) ? rb[0] * dc : rb[k] * scale;
            const double ai = (k == 0) ? 0.0 : -rb[n - k] * scale;
            const double v1r = ar * cr - ai * ci, v1i = ar * ci + ai * cr;
            const double c2r = r2 * (cr - ci), c2i = r2 * (cr + ci);
            const double br = rb[k + N] * scale, bi = -rb[N - k] * scale;
            const double v2r = br * c2r - bi * c2i, v2i = br * c2i + bi * c2r;
            const double2 sp = __ldg(tw + 2 * k);
            const double sr = sp.x, si = -sp.y;
            const double dr = v1r - v2r, di = v1i - v2i;
            const double qr = sr * dr - si * di, qi = sr * di + si * dr;
            cb[pad8(brev(k, logn - 1))] = make_double2(0.5 * (v1r + v2r - qi), 0.5 * (v1i + v2i + qr));
        }
    }
    __syncthreads();
    fft_from_bitreversed<double, true>(cb, N, logn - 1, P.tw2n, 2);
    for (int j = tid; j < n; j += nt) {
        const int q = (j & 1) ? (n - 1 - (j >> 1)) : (j >> 1);
        const double2 w = cb[pad8(q >> 1)];
        o[j] = (q & 1) ? w.y : w.x;
    }
}

/// Threads per CTA: one radix-8 group of the n-point FFT per thread (n / 8),
/// 128..512 (measured: n / 16 and n / 4 are 10-35% slower at n = 2048).
int nfst_threads(int n) { return std::min(512, std::max(128, n / 8)); }

std::size_t nfst_smem_bytes(int n) {
    return static_cast<std::size_t>(cb_len(n)) * sizeof(double2) + (n + 2 * kHalo + 8 + 40) * sizeof(double);
}

} // namespace

bool nfst_supported(std::size_t n, int taps) {
    return is_pow2(n) && n >= 128 && n <= 8192 && taps <= 57 && nfst_smem_bytes(static_cast<int>(n)) <= 227 * 1024;
}

cudaError_t nfst_apply(const double* in, double* out, std::size_t batch, const FastPlanDev& P, int* flag,
                       bool inverse, cudaStream_t stream) {
    if (batch == 0) return cudaSuccess;
    if (!nfst_supported(P.n, P.taps)) return cudaErrorInvalidValue;
    const std::size_t smem = nfst_smem_bytes(P.n);
    auto kern = inverse ? nfst_inverse_kernel : nfst_forward_kernel;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(batch), nfst_threads(P.n), smem, stream>>>(in, out, P, flag);
    return cudaGetLastError();
}

} // namespace dctp::dev
