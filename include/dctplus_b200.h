/*
 * dctplus_b200 — C ABI of the B200-native batched Fast DCT+ (arXiv 2409.08970).
 *
 * This is the drop-in boundary for the reference's hot path: the transform
 * construction and apply API of proj/include/dctplus/fast_transform.hpp.
 * Plain pointers, sizes and status codes only; no C++ or torch types.  The
 * C++ mirror of the reference API (include/dctplus_b200/dctplus.hpp) and the
 * Python package (paper_2409_08970_b200) both sit on this header.
 *
 * Conventions
 *  - Every function returns a dctp_status; on failure dctp_last_error()
 *    returns the message of the calling thread's last error.  The status
 *    codes map 1:1 to the exception classes the reference throws
 *    (fast_transform.hpp:52-53,266-276; graph.hpp:95-108; spectral.hpp:190,
 *    :306-311; fast_transform.hpp:67-68).
 *  - Vertex indices are 1-based, as in RankOneUpdate (graph.hpp:87-114).
 *  - Signals are rows: batch x n, row-major, each signal contiguous (the
 *    reference's std::vector per signal).  Output coefficients are in
 *    ascending-eigenvalue slot order (proj/README.md:82).
 *  - *_f64 / *_f32 entry points take DEVICE pointers on the plan's device and
 *    run asynchronously on `stream` (a cudaStream_t, NULL = legacy default).
 *    Non-finite inputs raise a device flag; dctp_plan_sync_check() waits for
 *    the stream and returns DCTP_DOMAIN_ERROR if it was raised (the
 *    reference's check_signal, fast_transform.hpp:271-276).
 *  - *_host_* entry points take HOST pointers and are synchronous (they copy
 *    in, transform and copy out; pinned memory gives full PCIe bandwidth).
 *  - Plans are immutable after creation and may be used concurrently from
 *    any host thread on any stream of the plan's device.
 */
#ifndef DCTPLUS_B200_H
#define DCTPLUS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum dctp_status {
    DCTP_OK = 0,
    DCTP_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    DCTP_DOMAIN_ERROR = 2,     /* std::domain_error (non-finite input, pole collision) */
    DCTP_RUNTIME_ERROR = 3,    /* std::runtime_error (secular non-convergence) */
    DCTP_LOGIC_ERROR = 4,      /* std::logic_error (repeated path eigenvalues) */
    DCTP_CUDA_ERROR = 5        /* CUDA failure (no reference counterpart) */
} dctp_status;

typedef enum dctp_update_kind {
    DCTP_SELF_LOOP = 0,  /* RankOneUpdate::self_loop(i, w):     v = e_i        */
    DCTP_EDGE_DELTA = 1, /* RankOneUpdate::edge_delta(i, j, w): v = e_i - e_j  */
    DCTP_GENERAL = 2     /* extension: caller-supplied v of length n (config 5) */
} dctp_update_kind;

typedef struct dctp_plan dctp_plan;
typedef struct dctp_ensemble dctp_ensemble;
typedef struct dctp_chain dctp_chain;

/* Message of the calling thread's last failure ("" if none). */
const char* dctp_last_error(void);

/* Library version string and the CUDA architecture it was built for. */
const char* dctp_version(void);

/* --- DctPlusPlan (fast_transform.hpp:43-302) ------------------------------ */

/* DctPlusPlan(n, update, epsilon, tau) (fast_transform.hpp:45).  For
 * DCTP_GENERAL, `v` holds n doubles; otherwise it is ignored (may be NULL).
 * `device` is the CUDA ordinal the plan's constants are uploaded to; a
 * negative device builds a host-only plan (setup vectors and basis only —
 * the apply entry points then return DCTP_INVALID_ARGUMENT). */
int dctp_plan_create(size_t n, int kind, size_t i, size_t j, double rho, const double* v,
                     double epsilon, double tau, int device, dctp_plan** out);
int dctp_plan_destroy(dctp_plan* plan);

/* size(), epsilon(), slow_path() (fast_transform.hpp:136-143) and the
 * kept / active counts of the secular subproblem. */
int dctp_plan_info(const dctp_plan* plan, size_t* n, double* epsilon, int* slow_path,
                   size_t* n_kept, size_t* n_active, int* device);

/* Forward route of the plan's fp64 apply (no reference counterpart; the
 * reference picks its route in the constructor, fast_transform.hpp:86-133):
 * *nfst = 1 when forward() runs the NFST fast route (the reference's own
 * algorithm, nfst.cu), 0 for an exact route; *probe_gap = max-norm relative
 * gap between the NFST and exact routes on the creation probe (0 when the
 * NFST route is unavailable for the plan). */
int dctp_plan_route(const dctp_plan* plan, int* nfst, double* probe_gap);

/* Int8 tensor-core products (no reference counterpart): *slices = the number
 * of int8 digits per operand the fp64 dense products of length-n rows use on
 * the tcgen05 kind::i8 path (ozaki.cu; slices (slices + 1) / 2 integer GEMMs
 * per product), 0 when they run on the DMMA fp64 tensor cores.  The dense
 * route (forward/inverse of dense plans such as config 5, forward_nmvp,
 * inverse(fast = false)) and the rank-k chain apply take this path in fp64. */
int dctp_ozaki_slices(size_t n, int* slices);

/* Host copies of the setup vectors, n doubles each (any pointer may be NULL):
 * lambda(), mu(), the deflated z, per-slot normalisers a, per-slot signs sigma
 * (factorization(), cauchy.hpp:111-119). */
int dctp_plan_setup(const dctp_plan* plan, double* lambda, double* mu, double* z, double* a,
                    double* sigma);

/* Slot map (spectral.hpp:322-325): passthrough[s] in {0,1}, idx[s]. */
int dctp_plan_slots(const dctp_plan* plan, int* passthrough, int64_t* idx);

/* The active subproblem of PerturbedSpectrum (spectral.hpp:330-338): *k = the
 * number of kept (non-deflated) indices; sub_lambda, sub_z, sub_mu (k doubles
 * each, any may be NULL) and *rho — factorization().spec. */
int dctp_plan_subproblem(const dctp_plan* plan, size_t* k, double* sub_lambda, double* sub_z, double* sub_mu,
                         double* rho);

/* Dense basis X (n x n row-major, signed) — basis() (fast_transform.hpp:142),
 * rebuilt on the host on demand. */
int dctp_plan_basis(const dctp_plan* plan, double* x);

/* Batched forward (fast_transform.hpp:163-190) and inverse (:218-255) on
 * device rows. in/out: batch x n.  in and out must not alias. */
int dctp_forward_f64(const dctp_plan* plan, const double* d_in, double* d_out, size_t batch, void* stream);
int dctp_forward_f32(const dctp_plan* plan, const float* d_in, float* d_out, size_t batch, void* stream);
int dctp_inverse_f64(const dctp_plan* plan, const double* d_in, double* d_out, size_t batch, void* stream);
int dctp_inverse_f32(const dctp_plan* plan, const float* d_in, float* d_out, size_t batch, void* stream);

/* Waits for `stream`; DCTP_DOMAIN_ERROR if any input since the last check was
 * non-finite (then clears the flag). */
int dctp_plan_sync_check(const dctp_plan* plan, void* stream);

/* Dense routes with the materialised basis X (built on first use, n^2
 * doubles twice on the device): forward_nmvp = X^T s (fast_transform.hpp:
 * 199-214) and inverse(p, fast = false) = X p (:218-260), fp64 tensor cores. */
int dctp_forward_nmvp_f64(const dctp_plan* plan, const double* d_in, double* d_out, size_t batch, void* stream);
int dctp_forward_nmvp_f32(const dctp_plan* plan, const float* d_in, float* d_out, size_t batch, void* stream);
int dctp_inverse_nmvp_f64(const dctp_plan* plan, const double* d_in, double* d_out, size_t batch, void* stream);
int dctp_inverse_nmvp_f32(const dctp_plan* plan, const float* d_in, float* d_out, size_t batch, void* stream);

/* Synchronous host-buffer variants (H2D, forward/inverse, D2H). */
int dctp_forward_host_f64(const dctp_plan* plan, const double* h_in, double* h_out, size_t batch);
int dctp_inverse_host_f64(const dctp_plan* plan, const double* h_in, double* h_out, size_t batch);
int dctp_forward_host_f32(const dctp_plan* plan, const float* h_in, float* h_out, size_t batch);
int dctp_inverse_host_f32(const dctp_plan* plan, const float* h_in, float* h_out, size_t batch);
int dctp_forward_nmvp_host_f64(const dctp_plan* plan, const double* h_in, double* h_out, size_t batch);
int dctp_forward_nmvp_host_f32(const dctp_plan* plan, const float* h_in, float* h_out, size_t batch);
int dctp_inverse_nmvp_host_f64(const dctp_plan* plan, const double* h_in, double* h_out, size_t batch);
int dctp_inverse_nmvp_host_f32(const dctp_plan* plan, const float* h_in, float* h_out, size_t batch);

/* --- PrunedEnsemblePlan (fast_transform.hpp:338-454) ----------------------- */

/* PrunedEnsemblePlan(n, updates, cp, threshold, epsilon) (:343), 1 <= cp <= n.
 * The K updates are given as parallel arrays; vs holds K*n doubles for
 * DCTP_GENERAL members (may be NULL otherwise). */
int dctp_ensemble_create(size_t n, size_t k, const int* kinds, const size_t* is, const size_t* js,
                         const double* rhos, const double* vs, size_t cp, double threshold,
                         double epsilon, int device, dctp_ensemble** out);
int dctp_ensemble_destroy(dctp_ensemble* ens);
/* ensemble_size() (= K + 1) and member(r), r in 1..K (:380-381). */
int dctp_ensemble_info(const dctp_ensemble* ens, size_t* n, size_t* ensemble_size);
int dctp_ensemble_member(const dctp_ensemble* ens, size_t r, const dctp_plan** member);

/* forward_all (:396-439): out is batch x (K+1) x n; set 0 is the shared DCT.
 * Signals whose path quadratic form is <= threshold take the pruned branch
 * when cp < n (first cp coefficients of every set, the rest zero). */
int dctp_ensemble_forward_all_f64(const dctp_ensemble* ens, const double* d_in, double* d_out,
                                  size_t batch, void* stream);
int dctp_ensemble_forward_all_f32(const dctp_ensemble* ens, const float* d_in, float* d_out,
                                  size_t batch, void* stream);
/* forward_all with the rest of Result (:383-387): bounds (batch x (K+1),
 * truncation-error bound per set, 0 on the full branch) and pruned (batch,
 * 1 = pruned branch); either may be NULL. */
int dctp_ensemble_forward_all_pruned_f64(const dctp_ensemble* ens, const double* d_in, double* d_out,
                                         double* d_bounds, unsigned char* d_pruned, size_t batch, void* stream);
int dctp_ensemble_forward_all_pruned_f32(const dctp_ensemble* ens, const float* d_in, float* d_out,
                                         float* d_bounds, unsigned char* d_pruned, size_t batch, void* stream);
int dctp_ensemble_sync_check(const dctp_ensemble* ens, void* stream);
/* rdo_select (fast_transform.hpp:472-496, l1 cost) for a batch of device rows:
 * index (batch, int) of the least-l1 set per signal (ties to the lower index),
 * chosen (batch x n) that set's coefficients, pruned (batch) the branch; the
 * outputs may be NULL (not both chosen and index). */
int dctp_ensemble_rdo_select_f64(const dctp_ensemble* ens, const double* d_in, double* d_chosen, int* d_index,
                                 unsigned char* d_pruned, size_t batch, void* stream);
int dctp_ensemble_rdo_select_f32(const dctp_ensemble* ens, const float* d_in, float* d_chosen, int* d_index,
                                 unsigned char* d_pruned, size_t batch, void* stream);
/* Host-buffer forward_all with bounds / pruned (synchronous; NULL-able outputs). */
int dctp_ensemble_forward_all_pruned_host_f64(const dctp_ensemble* ens, const double* h_in, double* h_out,
                                              double* h_bounds, unsigned char* h_pruned, size_t batch);
int dctp_ensemble_forward_all_pruned_host_f32(const dctp_ensemble* ens, const float* h_in, float* h_out,
                                              float* h_bounds, unsigned char* h_pruned, size_t batch);
int dctp_ensemble_forward_all_host_f32(const dctp_ensemble* ens, const float* h_in, float* h_out, size_t batch);
int dctp_ensemble_forward_all_host_f64(const dctp_ensemble* ens, const double* h_in, double* h_out, size_t batch);

/* --- rank-k chains (cauchy.hpp:159-231) ------------------------------------ */

/* compose_rank_k(base, updates, tau) (cauchy.hpp:175-216): k >= 1 rank-one
 * updates (parallel arrays as in dctp_ensemble_create) applied in order on top
 * of a base spectrum: base_lambda (n, ascending) and base_u (n x n row-major,
 * column k = eigenvector k), or both NULL for path_spectrum(n)
 * (spectral.hpp:48-68).  The composition runs on the host and reproduces the
 * reference's final basis and eigenvalues bit for bit; a failing stage r
 * returns DCTP_RUNTIME_ERROR with "compose_rank_k: stage r: ..." as the
 * reference throws it.  device < 0: host-only chain (no apply). */
int dctp_chain_create(size_t n, size_t k, const int* kinds, const size_t* is, const size_t* js,
                      const double* rhos, const double* vs, const double* base_lambda, const double* base_u,
                      double tau, int device, dctp_chain** out);
int dctp_chain_destroy(dctp_chain* chain);
int dctp_chain_info(const dctp_chain* chain, size_t* n, size_t* stages);
/* ChainedFactorization::mu (n, ascending) and ::x (n x n row-major, signed);
 * either may be NULL. */
int dctp_chain_spectrum(const dctp_chain* chain, double* mu, double* x);
/* Stage r (0-based) of ::stages: base_vals (n), spec.mu (n), sigma (n),
 * spec.slots (passthrough, idx; n each), number of deflation rotations; all
 * NULL-able. */
int dctp_chain_stage(const dctp_chain* chain, size_t r, double* base_vals, double* mu, double* sigma,
                     int* passthrough, int64_t* idx, size_t* n_rotations);
/* chain_forward (cauchy.hpp:218-231) for batch x n device rows: out = in X. */
int dctp_chain_forward_f64(const dctp_chain* chain, const double* d_in, double* d_out, size_t batch, void* stream);
int dctp_chain_forward_f32(const dctp_chain* chain, const float* d_in, float* d_out, size_t batch, void* stream);
int dctp_chain_sync_check(const dctp_chain* chain, void* stream);
int dctp_chain_forward_host_f64(const dctp_chain* chain, const double* h_in, double* h_out, size_t batch);
int dctp_chain_forward_host_f32(const dctp_chain* chain, const float* h_in, float* h_out, size_t batch);

/* --- batched trig kernels (trig.hpp:95-110), orthonormal ------------------ */
int dctp_dct2_f64(size_t n, const double* d_in, double* d_out, size_t batch, int device, void* stream);
int dctp_idct2_f64(size_t n, const double* d_in, double* d_out, size_t batch, int device, void* stream);
int dctp_dct2_f32(size_t n, const float* d_in, float* d_out, size_t batch, int device, void* stream);
/* Host-buffer form (TrigPlan::execute, trig.hpp:95-110): `batch` rows of n
 * doubles through the GPU kernels, synchronous.  inverse = 0: dct2, 1: idct2. */
int dctp_trig_host_f64(int inverse, size_t n, const double* h_in, double* h_out, size_t batch, int device);
int dctp_idct2_f32(size_t n, const float* d_in, float* d_out, size_t batch, int device, void* stream);

/* --- profiling: CUDA-event timing of every kernel launch ---------------- */
/* When enabled, each kernel the library launches is bracketed by two CUDA
 * events on its stream.  dctp_profile_summary() waits for them and writes
 * {"kernel": [launches, total_ms], ...} as JSON into buf. */
int dctp_profile_enable(int on);
int dctp_profile_reset(void);
int dctp_profile_summary(char* buf, size_t len);

/* --- seeded inputs: signal.hpp Rng / gen_ar_signal, bench.hpp mix_seed ---- */
uint64_t dctp_mix_seed(uint64_t seed, size_t size, size_t kind);
/* dist 0: Rng::gaussian(), 1: Rng::uniform(), 2: rows of gen_ar_signal(n, r),
 * 3: 2*uniform()-1, 4: 2-D separable AR(1) rows (fields of n x n, rho = r). */
int dctp_fill_signals(uint64_t seed, int dist, double r, size_t n, size_t rows, double* out);

#ifdef __cplusplus
}
#endif

#endif /* DCTPLUS_B200_H */
