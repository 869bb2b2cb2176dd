// Host-visible launchers of the sm_100a kernels (no CUDA types leak beyond
// cudaStream_t).  Implemented in dct.cu / cauchy.cu; called by plan.cpp.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include <cuda_runtime_api.h>

namespace dctp::dev {

/// Twiddle tables of one power-of-two length n (N = n/2 complex points),
/// interleaved (cos, sin) in T, device-resident.
template <class T>
struct Twiddles {
    const T* fft = nullptr;   // e^{-2 pi i k / N},      k < N/2
    const T* split = nullptr; // e^{-2 pi i k / n},      k < N
    const T* rot = nullptr;   // e^{-i pi k / (2n)},     k <= N
    const T* cos4n = nullptr; // cos(pi m / (2n)), m < 4n (direct kernels, any n)
};

/// Index/value list for a scattered copy dst[b*ld + to[e]] = sign[e] * src[from[e]].
template <class T>
struct Emit {
    const int* to = nullptr;   // >= 0: index into the row of `out`; < 0: index -to-1 into the row of `alt`
    const int* from = nullptr;
    const T* sign = nullptr;
    int count = 0;
    T* alt = nullptr;          // second target (the compacted kept coefficients), row stride ld_alt
    std::size_t ld_alt = 0;
};

/// Whether the DCT-II/III kernels take rows of length n (the row lives in
/// shared memory: powers of two up to 8192 in fp64 / 16384 in fp32, other
/// lengths up to 14528 / 29056).
bool dct_supported(std::size_t n, bool f64);

/// Forward DCT-II of `batch` rows of length n (orthonormal, U^T s):
///   hat[b*ld_hat + k]     = shat_k          (if hat != nullptr)
///   out[b*ld_out + to[e]] = sign[e] * shat_{from[e]}   for each emit entry
/// Non-finite input samples set *flag (the domain_error of check_signal).
template <class T>
cudaError_t dct2_rows(const T* in, std::size_t ld_in, T* hat, std::size_t ld_hat, T* out,
                      std::size_t ld_out, Emit<T> emit, std::size_t n, std::size_t batch,
                      Twiddles<T> tw, int* flag, cudaStream_t stream);

/// int8 slices of u written by the folded DCT kernel instead of u itself
/// (fp64): the int8 GEMM's A image (ozaki.cu layout: tiles of tile_rows rows,
/// nch 64-byte chunks, S slices) and per-row exponents.
struct FoldSlices {
    int8_t* sl = nullptr;
    int* expo = nullptr;
    int S = 0, nch = 0, tile_rows = 0;
    const int* map = nullptr; // idct_rows: the K gathered columns of p to slice (the folded inverse's W slots)
    int K = 0;
    // fp32: the same values leave as the bf16x3 GEMM's A image instead (hi /
    // lo bf16 halves, tc_bf16x3_a_bytes layout) — no u round trip / split pass
    unsigned char* bf = nullptr;
};

/// Folded forward of antisymmetric plans: rows of 2n samples x; writes
/// u_j = x_j - x_{2n-1-j} (n per row) to `u` (or, with fs.sl, its int8
/// slices) and emits the DCT-II (length n) of y_j = x_j + x_{2n-1-j} through
/// `emit`.
template <class T>
cudaError_t dct2_fold_rows(const T* in, std::size_t ld_in, T* u, std::size_t ld_u, T* out, std::size_t ld_out,
                           Emit<T> emit, std::size_t n, std::size_t batch, Twiddles<T> tw, int* flag,
                           cudaStream_t stream, FoldSlices fs = {});

/// Inverse (DCT-III, orthonormal, U d) of rows d; before the transform
///   d[to[e]] = sign[e] * p[b*ld_p + from[e]]  (the pass-through slots).
template <class T>
cudaError_t idct_rows(const T* d, std::size_t ld_d, const T* p, std::size_t ld_p, Emit<T> emit,
                      T* out, std::size_t ld_out, std::size_t n, std::size_t batch,
                      Twiddles<T> tw, int* flag, cudaStream_t stream, FoldSlices fs = {});

/// One Cauchy stage (SIMT, entries generated on the fly from fp64 gaps):
///   out[b*ld_out + dst[c]] = cscale[c] * sum_r rscale[r] * in[b*ld_in + src[r]] / (x[r] - y[c])
struct CauchyStage {
    const int* src;       // R
    const double* x;      // R
    const void* rscale;   // R, T
    const int* dst;       // C
    const double* y;      // C
    const void* cscale;   // C, T
    int rows;             // R
    int cols;             // C
    std::int64_t out_offset; // element offset of this stage's output within a row block
    int src_contig;       // 1: src[r] == r (rows of `in` already compacted); enables 16-byte loads
};

template <class T>
cudaError_t cauchy_rows(const T* in, std::size_t ld_in, T* out, std::size_t ld_out,
                        const CauchyStage* stages_dev, int num_stages, int max_rows, int max_cols,
                        std::size_t batch, int* flag, cudaStream_t stream);

/// fp64 Cauchy stage on the tensor cores (cauchy_dmma.cu); same contract as
/// cauchy_rows<double>.
cudaError_t cauchy_rows_dmma(const double* in, std::size_t ld_in, double* out, std::size_t ld_out,
                             const CauchyStage* stages_dev, int num_stages, int max_cols, std::size_t batch,
                             int* flag, cudaStream_t stream);

/// Constants of the fused small-plan forward kernel (fused_small.cu).
/// Generic plans: the Cauchy stage multiplies the kept DCT coefficients by
/// tmat = T (A x K, row c = output column); pass-through slots copy the DCT
/// coefficient pass_src scaled by pass_coef (= sigma).  Folded plans (every
/// kept DCT index odd): the Cauchy stage multiplies u_j = x_j - x_{n-1-j}
/// (K = n/2) by tmat = W^T, W = D_odd^T T (plus sigma D rows for odd
/// pass-through slots), and the length-n/2 DCT-II of y_j = x_j + x_{n-1-j}
/// feeds the even pass-through slots (pass_coef = sigma / sqrt 2).
struct SmallPlanDev {
    const int* act_slot;     // A: output slot of column c
    const double* tmat;      // A x K, row-major
    const int* kept_idx;     // K: DCT index of each kept coefficient (generic only)
    const int* pass_src;     // n_pass: index into the length-L DCT coefficients
    const int* pass_slot;    // n_pass: output slot
    const double* pass_coef; // n_pass: multiplier
    const double* fft_tw;    // L/2 complex e^{-2 pi i m / (L/2)}
    const double* split_tw;  // L/2 complex e^{-2 pi i k / L}
    const double* rot_tw;    // L/2+1 complex e^{-i pi k / 2L}
    int n, K, A, n_pass, fold;
    unsigned long long* timers; // DCTP_DEBUG_MODE & 4: producer phase cycle counters (7)
    int debug; // development knob (DCTP_DEBUG_MODE bits): 1 = skip the DCT work, 2 = skip the DMMA work
};

/// Pruned progressive mode (fast_transform.hpp:396-439, c_p < n) applied in
/// place to a batch already transformed in full (`out`, batch x (K+1) x n);
/// blocks = K x n x c_p ([UL_r; HL_r]).  c_p >= n: only the optional outputs
/// (bounds 0, pruned = path quadratic form <= threshold).
template <class T>
cudaError_t ensemble_prune(const T* in, T* out, const T* blocks, std::size_t n, std::size_t cp, int members,
                           double threshold, std::size_t batch, T* bounds, unsigned char* pruned,
                           cudaStream_t stream);

/// rdo_select (fast_transform.hpp:472-496) over forward_all output rows
/// (batch x sets x n): index of the least-l1 set per signal (ties to the
/// lower index) and, if `chosen` is set, that set's coefficients (batch x n).
template <class T>
cudaError_t rdo_select_rows(const T* coeffs, std::size_t n, int sets, std::size_t batch, T* chosen, int* index,
                            cudaStream_t stream);

/// Generic plans: power-of-two 16 <= n <= 512, K <= 128, A <= 128.  Folded
/// plans: power-of-two 64 <= n <= 256 and at most 128 Cauchy columns.
/// C[M x N] = A[M x K] * B[K x N], fp32 row-major (K % 16 == 0, N and the
/// leading dimensions multiples of 4, 16-byte aligned); raises flag bit 0 if
/// column 0 of a row is non-finite (the progressive DC coefficient).
bool sgemm_rows_supported(int K, int N, int lda, int ldb, std::size_t ldc, const void* A, const void* B, const void* C);
cudaError_t sgemm_rows(const float* A, int lda, const float* B, int ldb, float* C, std::size_t ldc, std::size_t M,
                       int N, int K, int* flag, cudaStream_t stream, const int* col_map = nullptr);

/// Signed DCT-domain rows of a plan's basis (row s = sigma_s y_s, n x ld) and
/// an n x n transpose: with idct_rows these materialise X^T and X on the device.
cudaError_t basis_coefficients(int n, std::size_t ld, const double* z, const double* lambda, const double* nu,
                               const int* pass_idx, const double* a, const double* sigma, double* y,
                               cudaStream_t stream, int rows = -1);
cudaError_t transpose_square(const double* in, std::size_t ld_in, double* out, std::size_t ld_out, int n,
                             cudaStream_t stream);

/// v[b, c] = sum_k in[b, a_map ? a_map[k] : k] bt[c, k] on the DMMA tensor
/// cores (bt row-major, 16-byte aligned rows, ld_bt even), stored to
/// out[b, col_map ? col_map[c] : c], or — with fold_add — unfolded:
/// out[b, c] = add[b, c] + v, out[b, 2N-1-c] = add[b, c] - v.  The rank-k
/// chain apply, the dense routes, and the folded route's W products.
template <class T>
cudaError_t rows_by_basis(const T* in, std::size_t ld_in, const double* bt, std::size_t ld_bt, int K, int N, T* out,
                          std::size_t ld_out, std::size_t batch, int* flag, cudaStream_t stream,
                          const int* col_map = nullptr, const int* a_map = nullptr, const T* fold_add = nullptr,
                          std::size_t ld_add = 0);

/// fp64 products on the int8 tcgen05 tensor cores (ozaki.cu).  Operands are
/// sliced first: each row r of `in` (rows x K, row stride ld; columns
/// gathered through a_map if given) becomes `slices` int8 digits with a
/// power-of-two row exponent expo[r], written in the GEMM's tile image for
/// tiles of `tile_rows` rows (128 for the A side, ozaki_tile_n(slices) for
/// the B side), rows zero-padded to a multiple of pad_rows (ozaki_pad_m() /
/// ozaki_pad_n(slices)); non-finite samples raise flag bit 0.  Then
///   out[b, col_map ? col_map[c] : c] = sum_k a[b, k] bt[c, k]
/// (or unfolded with fold_add as in rows_by_basis) for M rows of a and N rows
/// of bt, accurate to ~1e-13 (6 slices) / ~3e-11 (5 slices) of the row
/// maxima.  K <= 16384.
int ozaki_tile_n(int slices);
int ozaki_pad_n(int slices);
int ozaki_pad_m();
std::size_t ozaki_slice_bytes(std::size_t rows, int K, int tile_rows, int slices, int pad_rows = 0);
template <class T>
cudaError_t ozaki_slice(const T* in, std::size_t ld, std::size_t rows, int K, const int* a_map, int tile_rows,
                        int slices, int8_t* sl, int* expo, int* flag, cudaStream_t stream, int pad_rows = 0);
/// Folded rows x (2L samples) -> the sliced K = 2L operand [y | u] (y_j =
/// x_j + x_{2L-1-j}, u_j = x_j - x_{2L-1-j}), one exponent per row; L % 4 == 0,
/// L <= 1024, 16-byte aligned rows.
cudaError_t ozaki_slice_fold(const double* in, std::size_t ld, std::size_t rows, int L, int tile_rows, int slices,
                             int8_t* sl, int* expo, int* flag, cudaStream_t stream, int pad_rows = 0);
/// Grouped product on the persistent CTA-pair kernel: output column tiles
/// (ozaki_group_tile(slices) columns each) below nt_split contract K columns
/// [0, k_split) of a and bt, the others [k_split, K) — two products with
/// different operand halves (the fold's D y and W u) in one launch, each
/// output row written by one kernel; col_map < 0 skips padding columns.
bool ozaki_grouped_supported();
int ozaki_group_tile(int slices);
cudaError_t ozaki_gemm_grouped(const int8_t* a_sl, const int* ea, const int8_t* b_sl, const int* eb, std::size_t M,
                               int N, int K, int slices, double* out, std::size_t ld_out, const int* col_map,
                               int nt_split, int k_split, cudaStream_t stream);
cudaError_t ozaki_gemm(const int8_t* a_sl, const int* ea, const int8_t* b_sl, const int* eb, std::size_t M, int N,
                       int K, int slices, double* out, std::size_t ld_out, const int* col_map, cudaStream_t stream,
                       const double* fold_add = nullptr, std::size_t ld_add = 0);

/// Constants of the NFST fast route (nfst.cu), the reference's own
/// DctPlusPlan::forward algorithm (fast_transform.hpp:94-133, 163-190;
/// nfst.hpp:100-164, 201-238) built on the host in double like the reference.
struct FastPlanDev {
    const double* hz;        // n: h_j z_j, h_j = (-1)^(j+1) / sin(j pi / n) (j >= 1)
    const double* ez;        // n: ext_row_j z_j (exterior slot), or nullptr
    const double* inv_phi;   // n: 1 / phi_hat(k) of the Gaussian kernel, [0] = 0
    const double* tw2n;      // n complex: e^{-2 pi i k / 2n}, k < n
    const double* rot;       // n/2 + 1 complex: e^{-i pi k / 2n}
    const int* pass_slot;    // n_pass
    const int* pass_src;     // n_pass
    const double* pass_sign; // n_pass
    const int* t_slot;       // R interior targets: output slot
    const int* t_lo;         // first grid point of the tap window (may be < 0)
    const double* t_p0;      // weight of tap 0
    const double* t_b;       // weight ratio of consecutive taps (w_t = P0 B^t C_t)
    const double* t_ca;      // -scale / (4 sin(n theta))
    const double* t_cb;      // scale / nu
    const double* ctab;      // {C_0, C_1, R_0, R_1, E}: C_t = exp(-alpha (t - hw)^2), R_t = C_{t+2} / C_t,
                             // E = exp(-8 alpha), alpha = h^2 / 4 tau (tap-weight recurrence)
    double z0, ext_scale;
    int n, logn, R, taps, hw, n_pass, ext_slot; // ext_slot < 0: no exterior row
};

bool nfst_supported(std::size_t n, int taps);
/// Forward (DctPlusPlan::forward) or inverse (inverse(p, ws, fast = true))
/// of `batch` contiguous rows of n doubles through the NFST route.
cudaError_t nfst_apply(const double* in, double* out, std::size_t batch, const FastPlanDev& P, int* flag,
                       bool inverse, cudaStream_t stream);

/// Per-graph setup on the GPU (setup.cu, compiled with -fmad=false): the
/// secular roots mu (k sorted distinct lam, nonzero z, zz = sum z^2; status
/// bit 0 = no convergence) and the normalisers a (status bit 1 = collision,
/// bit 2 = degenerate column), bit-identical to host/setup.hpp.
cudaError_t secular_roots_gpu(const double* lam, const double* z, int k, double rho, double zz, double* mu,
                              int* status, cudaStream_t stream);
cudaError_t normalisers_gpu(const double* lam, const double* z, int m, const double* mu, int k, double* a,
                            int* status, cudaStream_t stream);
/// Column signs of the materialised basis (spectral.hpp:30-37): for each of
/// `cols` rows of xt (row s = column s of X, n entries, stride ld), +1 / -1
/// making the largest-|.| entry positive, ties within 1e-12 relative to the
/// lowest index; written to sign[s].
cudaError_t column_signs_gpu(const double* xt, std::size_t ld, int n, int cols, double* sign, cudaStream_t stream);

/// C[M x N] = A[M x K] * B[K x N] in fp32 on the tcgen05 tensor cores
/// (kind::tf32, 3xTF32 split; tc_sgemm.cu): A row-major, B given as B^T =
/// bt_hi + bt_lo (N x K, row stride ldb; bt_hi TF32-representable), C
/// row-major (or column c stored at col_map[c], or unfolded with fold_add as
/// in rows_by_basis); A's columns optionally gathered through a_map; 16-byte aligned pointers,
/// K, lda, ldb, ldc multiples of 4.  Raises flag bit 0 if column 0 of a row
/// of the product is non-finite.
bool tc_sgemm3_supported(int K, int N, int lda, int ldb, std::size_t ldc, const void* A, const void* Bh,
                         const void* Bl, const void* C);
cudaError_t tc_sgemm3(const float* A, int lda, const float* bt_hi, const float* bt_lo, int ldb, float* C,
                      std::size_t ldc, std::size_t M, int N, int K, int* flag, cudaStream_t stream,
                      const int* col_map = nullptr, const int* a_map = nullptr, const float* fold_add = nullptr,
                      std::size_t ld_add = 0, const float* b_sw = nullptr);
/// B^T (hi, lo) rearranged into the kernel's shared-memory blocks (per
/// 256-row tile and 16-wide K chunk: hi then lo, SWIZZLE_64B), so each stage
/// of B arrives by one 32 KB TMA bulk copy (pass as b_sw).
std::vector<float> tc_swizzle_b(const float* bt_hi, const float* bt_lo, int N, int K, int ldb);

/// C[M x N] = A[M x K] B (fp32, row-major A and C) on the tcgen05 tensor cores
/// with the bf16x3 split (tc_bf16x3.cu): a persistent kernel whose B^T
/// column tile stays resident (K <= 128) or streams with A (larger K); b_sw
/// from tc_bf16x3_swizzle_b (B^T given in fp64, N x K, row stride ldb).  A's
/// columns optionally gathered through a_map; output plain, scattered
/// (col_map) or unfolded (fold_add, as in rows_by_basis; N % 4 == 0).  Raises
/// flag bit 0 if column 0 of a row is non-finite.
bool tc_bf16x3_supported(int K, int N, std::size_t ldc, const void* C, bool fold = false);
std::vector<uint16_t> tc_bf16x3_swizzle_b(const double* bt, int N, int K, int ldb);
cudaError_t tc_bf16x3(const float* A, int lda, const uint16_t* b_sw, float* C, std::size_t ldc, std::size_t M, int N,
                      int K, int* flag, int num_sms, cudaStream_t stream, const int* col_map = nullptr,
                      const int* a_map = nullptr, const float* fold_add = nullptr, std::size_t ld_add = 0,
                      const unsigned char* a_img = nullptr);
/// Bytes of the bf16x3 GEMM's A image for M rows of K columns (128-row tiles
/// x 32-column chunks x hi | lo x 128 rows x 64 B, SWIZZLE_64B rows) — what
/// the fp32 fold kernels write when FoldSlices::bf is set; pass it to
/// tc_bf16x3 as a_img (A and a_map are then unused).
std::size_t tc_bf16x3_a_bytes(std::size_t M, int K);

/// out[b, c] = sum_k in[b, k] xt[c, k] for n in {16, 32, 64, 128}: one CTA
/// per 32 signals, X^T staged in shared memory, m8n8k4 DMMA (small_dense.cu)
/// — the latency route of small plans at small batches.
bool small_dense_supported(std::size_t n, const void* in, std::size_t ld_in, const void* out, std::size_t ld_out);
cudaError_t small_dense_forward(const double* in, std::size_t ld_in, const double* xt, std::size_t ld_xt, double* out,
                                std::size_t ld_out, std::size_t n, std::size_t batch, int* flag, cudaStream_t stream);

bool fused_small_supported(std::size_t n, int K, int A);
bool fused_small_fold_supported(std::size_t n, int columns);
cudaError_t fused_small_forward(const double* in, double* out, std::size_t batch, const SmallPlanDev& P, int* flag,
                                int num_sms, cudaStream_t stream);

} // namespace dctp::dev
