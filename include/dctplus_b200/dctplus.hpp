// dctplus_b200/dctplus.hpp — C++ mirror of the reference's transform API
// (proj/include/dctplus/{graph,fast_transform}.hpp) over the C ABI in
// include/dctplus_b200.h.  Header-only; link with libdctplus_b200.so.
//
// Same class and function names, argument meaning and exception types as the
// reference, so a caller switches with
//     #include <dctplus_b200/dctplus.hpp>
//     namespace dctplus = dctplus_b200;
// Differences a caller can see:
//   * every apply runs on the GPU (plan `device`, default 0); the std::vector
//     overloads copy through pinned-or-pageable host memory synchronously;
//   * batched device-pointer entry points (forward_batch / inverse_batch /
//     forward_all_batch) take rows of signals and a cudaStream_t (as void*);
//   * RankOneUpdate::general(v, rho) extends the two reference update kinds;
//   * ChainedFactorization keeps x, mu and per-stage data; chain_forward runs
//     one product with x on the GPU (chain_forward_batch for device rows).
#ifndef DCTPLUS_B200_DCTPLUS_HPP
#define DCTPLUS_B200_DCTPLUS_HPP

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dctplus_b200.h"

namespace dctplus_b200 {

namespace detail {
inline void check(int status) {
    if (status == DCTP_OK) return;
    const std::string msg = dctp_last_error();
    switch (status) {
        case DCTP_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case DCTP_DOMAIN_ERROR: throw std::domain_error(msg);
        case DCTP_LOGIC_ERROR: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}
} // namespace detail

/// Rank-one Laplacian update L + rho v v^T (graph.hpp:87-114), 1-based vertices.
struct RankOneUpdate {
    enum class Kind { self_loop, edge_delta, general };

    Kind kind;
    double rho;
    std::size_t node_i = 0, node_j = 0; // 1-based
    std::vector<double> v;              // general direction (extension)

    static RankOneUpdate self_loop(std::size_t i, double w) {
        if (i < 1) throw std::invalid_argument("RankOneUpdate: node index is 1-based");
        if (w == 0.0) throw std::invalid_argument("RankOneUpdate: weight must be nonzero");
        return {Kind::self_loop, w, i, 0, {}};
    }
    static RankOneUpdate edge_delta(std::size_t i, std::size_t j, double w) {
        if (i < 1 || i >= j) throw std::invalid_argument("RankOneUpdate: need 1 <= i < j");
        if (w == 0.0) throw std::invalid_argument("RankOneUpdate: weight must be nonzero");
        return {Kind::edge_delta, w, i, j, {}};
    }
    static RankOneUpdate general(std::vector<double> dir, double rho) {
        if (rho == 0.0) throw std::invalid_argument("RankOneUpdate: weight must be nonzero");
        if (dir.empty()) throw std::invalid_argument("RankOneUpdate: empty direction");
        return {Kind::general, rho, 0, 0, std::move(dir)};
    }
    std::vector<double> direction(std::size_t n) const {
        if (kind == Kind::general) {
            if (v.size() != n) throw std::invalid_argument("RankOneUpdate: direction length mismatch");
            return v;
        }
        if (node_i > n || (kind == Kind::edge_delta && node_j > n))
            throw std::invalid_argument("RankOneUpdate: node index exceeds graph size");
        std::vector<double> out(n, 0.0);
        out[node_i - 1] = 1.0;
        if (kind == Kind::edge_delta) out[node_j - 1] = -1.0;
        return out;
    }
    int abi_kind() const {
        return kind == Kind::self_loop ? DCTP_SELF_LOOP : (kind == Kind::edge_delta ? DCTP_EDGE_DELTA : DCTP_GENERAL);
    }
};

/// Caller-owned result buffer, one per thread (fast_transform.hpp:35-38).
struct DctPlusWorkspace {
    std::vector<double> out;
};

/// Dense row-major matrix (matrix.hpp:14-60): what basis() returns.
class Matrix {
  public:
    Matrix() = default;
    Matrix(std::size_t rows, std::size_t cols, double fill = 0.0) : rows_(rows), cols_(cols), data_(rows * cols, fill) {}
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    double& operator()(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
    double operator()(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    /// flat row-major view (index i * cols + j), as round 1's basis() returned
    double operator[](std::size_t k) const { return data_[k]; }

  private:
    std::size_t rows_ = 0, cols_ = 0;
    std::vector<double> data_;
};

/// spectral.hpp:322-338: slot map entry and the perturbed spectrum.
struct SlotRef {
    bool passthrough;
    std::size_t idx;
};
struct PerturbedSpectrum {
    std::vector<double> mu; // full length, ascending
    std::vector<double> z;  // deflated (zeros at passed indices)
    std::vector<double> a;  // per slot; 1.0 for pass-through slots
    std::vector<SlotRef> slots;
    double rho = 0.0;
    std::vector<double> sub_lambda, sub_z, sub_mu; // active subproblem
};

/// cauchy.hpp:111-119: X = U diag(z) C(lambda, mu) diag(sigma .* a) with
/// pass-through columns.
struct CauchyFactorization {
    std::vector<double> lambda;
    PerturbedSpectrum spec;
    std::vector<double> sigma;
    std::size_t size() const { return lambda.size(); }
    double rho() const { return spec.rho; }
    const std::vector<double>& mu() const { return spec.mu; }
};

enum class TrigKind { dct2, idct2 };

/// TrigPlan (trig.hpp:32-116): the orthonormal DCT-II / its inverse of one
/// length; execute() runs the GPU kernels on host buffers.
class TrigPlan {
  public:
    TrigPlan(TrigKind kind, std::size_t len, int device = 0) : kind_(kind), len_(len), device_(device) {
        if (len < 1) throw std::invalid_argument("TrigPlan: length must be positive");
    }
    std::size_t size() const { return len_; }
    TrigKind kind() const { return kind_; }
    void execute(const double* in, double* out) const {
        detail::check(dctp_trig_host_f64(kind_ == TrigKind::idct2 ? 1 : 0, len_, in, out, 1, device_));
    }
    std::vector<double> operator()(const std::vector<double>& in) const {
        if (in.size() != len_) throw std::invalid_argument("TrigPlan: size mismatch");
        std::vector<double> out(len_);
        execute(in.data(), out.data());
        return out;
    }

  private:
    TrigKind kind_;
    std::size_t len_;
    int device_;
};

/// Fast DCT+ of one rank-one update of the path graph (fast_transform.hpp:43-302).
class DctPlusPlan {
  public:
    DctPlusPlan(std::size_t n, const RankOneUpdate& update, double epsilon, double tau = 1e-12, int device = 0)
        : update_(update) {
        if (update.kind == RankOneUpdate::Kind::general && update.v.size() != n)
            throw std::invalid_argument("RankOneUpdate: direction length mismatch");
        dctp_plan* h = nullptr;
        detail::check(dctp_plan_create(n, update.abi_kind(), update.node_i, update.node_j, update.rho,
                                       update.v.empty() ? nullptr : update.v.data(), epsilon, tau, device, &h));
        h_.reset(h, [](dctp_plan* p) { dctp_plan_destroy(p); });
        init();
    }

    std::size_t size() const { return n_; }
    double epsilon() const { return eps_; }
    const RankOneUpdate& update() const { return update_; }
    bool slow_path() const { return slow_; }
    int device() const { return device_; }
    /// true when the fp64 forward runs the NFST fast route (dctp_plan_route).
    bool nfst_route() const {
        int f = 0;
        detail::check(dctp_plan_route(h_.get(), &f, nullptr));
        return f != 0;
    }
    const std::vector<double>& lambda() const { return state_->fact.lambda; }
    const std::vector<double>& mu() const { return state_->fact.spec.mu; }
    /// The plan's factorization (fast_transform.hpp:141): lambda, the perturbed
    /// spectrum (mu, deflated z, a, slots, subproblem) and the column signs.
    const CauchyFactorization& factorization() const { return state_->fact; }
    /// The DCT-II plan of the plan's size (fast_transform.hpp:262).
    const TrigPlan& dct_plan() const { return state_->dct; }

    /// Dense basis X (n x n, row-major), columns signed by the largest-entry
    /// rule (fast_transform.hpp:142); built on the host on first use.
    const Matrix& basis() const {
        std::call_once(state_->basis_once, [this] {
            Matrix x(n_, n_);
            detail::check(dctp_plan_basis(h_.get(), x.data()));
            state_->basis = std::move(x);
        });
        return state_->basis;
    }

    DctPlusWorkspace make_workspace() const { return DctPlusWorkspace{std::vector<double>(n_)}; }

    const std::vector<double>& forward(const std::vector<double>& s, DctPlusWorkspace& ws) const {
        check_size(s);
        ws.out.resize(n_);
        detail::check(dctp_forward_host_f64(h_.get(), s.data(), ws.out.data(), 1));
        return ws.out;
    }
    std::vector<double> forward(const std::vector<double>& s) const {
        DctPlusWorkspace ws = make_workspace();
        return forward(s, ws);
    }
    /// The reference's dense X^T s; identical math, same GPU route.
    /// X^T s with the materialised basis (dense product on the GPU).
    const std::vector<double>& forward_nmvp(const std::vector<double>& s, DctPlusWorkspace& ws) const {
        check_size(s);
        ws.out.resize(n_);
        detail::check(dctp_forward_nmvp_host_f64(h_.get(), s.data(), ws.out.data(), 1));
        return ws.out;
    }
    std::vector<double> forward_nmvp(const std::vector<double>& s) const {
        DctPlusWorkspace ws = make_workspace();
        return forward_nmvp(s, ws);
    }

    /// fast: transposed Cauchy + DCT-III; otherwise the dense X p.
    const std::vector<double>& inverse(const std::vector<double>& p, DctPlusWorkspace& ws, bool fast = true) const {
        check_size(p);
        ws.out.resize(n_);
        detail::check(fast ? dctp_inverse_host_f64(h_.get(), p.data(), ws.out.data(), 1)
                           : dctp_inverse_nmvp_host_f64(h_.get(), p.data(), ws.out.data(), 1));
        return ws.out;
    }
    std::vector<double> inverse(const std::vector<double>& p, bool fast = true) const {
        DctPlusWorkspace ws = make_workspace();
        return inverse(p, ws, fast);
    }

    // ---- batched, device-resident (rows of n samples) ----------------------
    void forward_batch(const double* d_in, double* d_out, std::size_t batch, void* stream = nullptr) const {
        detail::check(dctp_forward_f64(h_.get(), d_in, d_out, batch, stream));
    }
    void forward_batch(const float* d_in, float* d_out, std::size_t batch, void* stream = nullptr) const {
        detail::check(dctp_forward_f32(h_.get(), d_in, d_out, batch, stream));
    }
    void inverse_batch(const double* d_in, double* d_out, std::size_t batch, void* stream = nullptr) const {
        detail::check(dctp_inverse_f64(h_.get(), d_in, d_out, batch, stream));
    }
    void inverse_batch(const float* d_in, float* d_out, std::size_t batch, void* stream = nullptr) const {
        detail::check(dctp_inverse_f32(h_.get(), d_in, d_out, batch, stream));
    }
    /// Waits for `stream`; throws std::domain_error if any input was non-finite.
    void sync_check(void* stream = nullptr) const { detail::check(dctp_plan_sync_check(h_.get(), stream)); }
    /// Batched host-buffer apply (pipelined H2D / kernels / D2H).
    void forward_host(const double* h_in, double* h_out, std::size_t batch) const {
        detail::check(dctp_forward_host_f64(h_.get(), h_in, h_out, batch));
    }
    void inverse_host(const double* h_in, double* h_out, std::size_t batch) const {
        detail::check(dctp_inverse_host_f64(h_.get(), h_in, h_out, batch));
    }

    const dctp_plan* handle() const { return h_.get(); }

  private:
    friend class PrunedEnsemblePlan;
    DctPlusPlan(const dctp_plan* borrowed, RankOneUpdate update) : update_(std::move(update)) {
        h_.reset(const_cast<dctp_plan*>(borrowed), [](dctp_plan*) {});
        init();
    }
    void check_size(const std::vector<double>& s) const {
        if (s.size() != n_) throw std::invalid_argument("DctPlusPlan: signal size mismatch");
    }
    /// Host copies of the setup (shared by copies of the plan object).
    struct State {
        CauchyFactorization fact;
        TrigPlan dct;
        std::once_flag basis_once;
        Matrix basis;
        State(std::size_t n, int device) : dct(TrigKind::dct2, n, device) {}
    };
    void init() {
        int slow = 0;
        detail::check(dctp_plan_info(h_.get(), &n_, &eps_, &slow, nullptr, nullptr, &device_));
        slow_ = slow != 0;
        state_ = std::make_shared<State>(n_, device_ < 0 ? 0 : device_);
        auto& f = state_->fact;
        f.lambda.resize(n_);
        f.spec.mu.resize(n_);
        f.spec.z.resize(n_);
        f.spec.a.resize(n_);
        f.sigma.resize(n_);
        detail::check(dctp_plan_setup(h_.get(), f.lambda.data(), f.spec.mu.data(), f.spec.z.data(),
                                      f.spec.a.data(), f.sigma.data()));
        std::vector<int> pass(n_);
        std::vector<int64_t> idx(n_);
        detail::check(dctp_plan_slots(h_.get(), pass.data(), idx.data()));
        f.spec.slots.resize(n_);
        for (std::size_t s = 0; s < n_; ++s) f.spec.slots[s] = {pass[s] != 0, static_cast<std::size_t>(idx[s])};
        std::size_t k = 0;
        detail::check(dctp_plan_subproblem(h_.get(), &k, nullptr, nullptr, nullptr, &f.spec.rho));
        f.spec.sub_lambda.resize(k);
        f.spec.sub_z.resize(k);
        f.spec.sub_mu.resize(k);
        detail::check(dctp_plan_subproblem(h_.get(), &k, f.spec.sub_lambda.data(), f.spec.sub_z.data(),
                                           f.spec.sub_mu.data(), nullptr));
    }

    RankOneUpdate update_;
    std::shared_ptr<dctp_plan> h_;
    std::shared_ptr<State> state_;
    std::size_t n_ = 0;
    double eps_ = 0.0;
    bool slow_ = false;
    int device_ = 0;
};

inline DctPlusPlan plan_dctplus(std::size_t n, const RankOneUpdate& u, double epsilon, double tau = 1e-12) {
    return DctPlusPlan(n, u, epsilon, tau);
}
inline std::vector<double> forward(const DctPlusPlan& plan, const std::vector<double>& s) { return plan.forward(s); }
inline std::vector<double> forward_nmvp(const DctPlusPlan& plan, const std::vector<double>& s) {
    return plan.forward_nmvp(s);
}
inline std::vector<double> inverse(const DctPlusPlan& plan, const std::vector<double>& p) { return plan.inverse(p); }

/// Scratch for PrunedEnsemblePlan::forward_all (fast_transform.hpp:323-336):
/// one workspace per member plus the shared-DCT buffer, and here the flat
/// K+1 sets the GPU call fills before they are split into Result::coeffs.
struct PrunedWorkspace {
    std::vector<DctPlusWorkspace> members;
    std::vector<double> sd;
    std::vector<double> flat;
};

/// Shared DCT + K Cauchy stages, progressive mode c_p = n (fast_transform.hpp:338-454).
class PrunedEnsemblePlan {
  public:
    static constexpr std::size_t kDenseMemberCutoff = 128;

    PrunedEnsemblePlan(std::size_t n, const std::vector<RankOneUpdate>& updates, std::size_t cp, double threshold,
                       double epsilon = 1e-12, int device = 0)
        : n_(n), cp_(cp), threshold_(threshold) {
        const std::size_t k = updates.size();
        std::vector<int> kinds(k);
        std::vector<std::size_t> is(k), js(k);
        std::vector<double> rhos(k), vs;
        bool any_general = false;
        for (std::size_t r = 0; r < k; ++r) {
            kinds[r] = updates[r].abi_kind();
            is[r] = updates[r].node_i;
            js[r] = updates[r].node_j;
            rhos[r] = updates[r].rho;
            any_general |= updates[r].kind == RankOneUpdate::Kind::general;
        }
        if (any_general) {
            vs.assign(k * n, 0.0);
            for (std::size_t r = 0; r < k; ++r)
                if (updates[r].kind == RankOneUpdate::Kind::general) {
                    const auto d = updates[r].direction(n);
                    std::copy(d.begin(), d.end(), vs.begin() + static_cast<std::ptrdiff_t>(r * n));
                }
        }
        dctp_ensemble* h = nullptr;
        detail::check(dctp_ensemble_create(n, k, kinds.data(), is.data(), js.data(), rhos.data(),
                                           any_general ? vs.data() : nullptr, cp, threshold, epsilon, device, &h));
        h_.reset(h, [](dctp_ensemble* e) { dctp_ensemble_destroy(e); });
        for (std::size_t r = 1; r <= k; ++r) {
            const dctp_plan* m = nullptr;
            detail::check(dctp_ensemble_member(h_.get(), r, &m));
            members_.push_back(DctPlusPlan(m, updates[r - 1]));
        }
    }

    std::size_t size() const { return n_; }
    std::size_t keep_count() const { return cp_; }
    double threshold() const { return threshold_; }
    std::size_t ensemble_size() const { return members_.size() + 1; }
    const DctPlusPlan& member(std::size_t r) const { return members_.at(r - 1); }

    struct Result {
        bool pruned = false;
        std::vector<std::vector<double>> coeffs; // one vector per ensemble member
        std::vector<double> bounds;              // truncation-error bound per member (0 on the full branch)
    };

    PrunedWorkspace make_workspace() const {
        PrunedWorkspace ws;
        for (const auto& m : members_) ws.members.push_back(m.make_workspace());
        ws.sd.resize(n_);
        ws.flat.resize(ensemble_size() * n_);
        return ws;
    }

    /// fast_transform.hpp:396-439: res.coeffs[r] (K + 1 sets, set 0 = the
    /// shared DCT), res.bounds, res.pruned; reuses ws and res's storage.
    void forward_all(const std::vector<double>& s, PrunedWorkspace& ws, Result& res) const {
        if (s.size() != n_) throw std::invalid_argument("pruned_forward_all: size mismatch");
        const std::size_t sets = ensemble_size();
        ws.flat.resize(sets * n_);
        res.coeffs.resize(sets);
        res.bounds.assign(sets, 0.0);
        unsigned char pruned = 0;
        detail::check(dctp_ensemble_forward_all_pruned_host_f64(h_.get(), s.data(), ws.flat.data(),
                                                                res.bounds.data(), &pruned, 1));
        res.pruned = pruned != 0;
        for (std::size_t r = 0; r < sets; ++r)
            res.coeffs[r].assign(ws.flat.begin() + static_cast<std::ptrdiff_t>(r * n_),
                                 ws.flat.begin() + static_cast<std::ptrdiff_t>((r + 1) * n_));
        ws.sd.assign(res.coeffs[0].begin(), res.coeffs[0].end());
    }

    Result forward_all(const std::vector<double>& s) const {
        PrunedWorkspace ws = make_workspace();
        Result res;
        forward_all(s, ws, res);
        return res;
    }

    /// rows x (K+1) x n output, device-resident.
    void forward_all_batch(const float* d_in, float* d_out, std::size_t batch, void* stream = nullptr) const {
        detail::check(dctp_ensemble_forward_all_f32(h_.get(), d_in, d_out, batch, stream));
    }
    void forward_all_batch(const double* d_in, double* d_out, std::size_t batch, void* stream = nullptr) const {
        detail::check(dctp_ensemble_forward_all_f64(h_.get(), d_in, d_out, batch, stream));
    }
    void sync_check(void* stream = nullptr) const { detail::check(dctp_ensemble_sync_check(h_.get(), stream)); }

  private:
    std::size_t n_, cp_;
    double threshold_;
    std::shared_ptr<dctp_ensemble> h_;
    std::vector<DctPlusPlan> members_;
};

inline PrunedEnsemblePlan plan_pruned(std::size_t n, const std::vector<RankOneUpdate>& updates, std::size_t cp,
                                      double threshold, double epsilon = 1e-12) {
    return PrunedEnsemblePlan(n, updates, cp, threshold, epsilon);
}
inline PrunedEnsemblePlan::Result pruned_forward_all(const PrunedEnsemblePlan& plan, const std::vector<double>& s) {
    return plan.forward_all(s);
}

/// fast_transform.hpp:466-496: the member whose coefficients minimise `cost`
/// (default l1), ties to the lower index, per the threshold branch.
struct RdoChoice {
    std::size_t index = 0;
    std::vector<double> coeffs;
    bool pruned = false;
};

template <class Cost>
RdoChoice rdo_select(const PrunedEnsemblePlan& plan, const std::vector<double>& s, Cost cost) {
    PrunedEnsemblePlan::Result res = plan.forward_all(s);
    RdoChoice choice;
    choice.pruned = res.pruned;
    double best = cost(res.coeffs[0]);
    for (std::size_t r = 1; r < res.coeffs.size(); ++r) {
        const double c = cost(res.coeffs[r]);
        if (c < best) {
            best = c;
            choice.index = r;
        }
    }
    choice.coeffs = std::move(res.coeffs[choice.index]);
    return choice;
}

inline RdoChoice rdo_select(const PrunedEnsemblePlan& plan, const std::vector<double>& s) {
    return rdo_select(plan, s, [](const std::vector<double>& c) {
        double a = 0.0;
        for (double v : c) a += std::abs(v);
        return a;
    });
}

/// bench.hpp:99-108: the `quantile` of the path quadratic form over `trials`
/// AR(r) signals from Rng(mix_seed(seed, n, 9000)).
inline double calibrate_prune_threshold(std::size_t n, double r = 0.99, double quantile = 0.7,
                                        std::size_t trials = 512, std::uint64_t seed = 42) {
    std::vector<double> sig(n * trials);
    detail::check(dctp_fill_signals(dctp_mix_seed(seed, n, 9000), 2, r, n, trials, sig.data()));
    std::vector<double> q(trials);
    for (std::size_t t = 0; t < trials; ++t) {
        double acc = 0.0;
        for (std::size_t i = 0; i + 1 < n; ++i) {
            const double d = sig[t * n + i] - sig[t * n + i + 1];
            acc += d * d;
        }
        q[t] = acc;
    }
    std::sort(q.begin(), q.end());
    const std::size_t idx =
        std::min(trials - 1, static_cast<std::size_t>(quantile * static_cast<double>(trials - 1)));
    return q[idx];
}

// --- rank-k chains (cauchy.hpp:159-231) -------------------------------------

/// L = U diag(lambda) U^T (spectral.hpp:21-24); u row-major n x n, column k =
/// eigenvector k (the reference's Matrix u(j, k) flattened by rows).
struct SpectralBasis {
    std::vector<double> lambda;
    std::vector<double> u;
    bool path = false; // path_spectrum(n): rebuilt by the library with the reference's rounding
};

/// path_spectrum (spectral.hpp:48-68).
inline SpectralBasis path_spectrum(std::size_t n) {
    if (n < 2) throw std::invalid_argument("path_spectrum: need n >= 2");
    SpectralBasis b;
    const double pi = 3.14159265358979323846, nd = static_cast<double>(n), scale = std::sqrt(2.0 / nd);
    b.lambda.resize(n);
    b.u.resize(n * n);
    for (std::size_t k = 0; k < n; ++k) {
        b.lambda[k] = 2.0 - 2.0 * std::cos(static_cast<double>(k) * pi / nd);
        const double ck = (k == 0) ? 1.0 / std::sqrt(2.0) : 1.0;
        for (std::size_t j = 0; j < n; ++j)
            b.u[j * n + k] =
                ck * scale * std::cos(pi * static_cast<double>(k) * (2.0 * static_cast<double>(j) + 1.0) / (2.0 * nd));
    }
    b.lambda[0] = 0.0;
    b.path = true;
    return b;
}

/// compose_rank_k's result (cauchy.hpp:163-173): final signed basis x
/// (row-major), final eigenvalues mu, and the stage count.
class ChainedFactorization {
  public:
    ChainedFactorization(const SpectralBasis& base, const std::vector<RankOneUpdate>& updates, double tau = 1e-12,
                         int device = 0) {
        n = base.lambda.size();
        const std::size_t k = updates.size();
        std::vector<int> kinds(k);
        std::vector<std::size_t> is(k), js(k);
        std::vector<double> rhos(k), vs;
        bool any_general = false;
        for (std::size_t r = 0; r < k; ++r) {
            kinds[r] = updates[r].abi_kind();
            is[r] = updates[r].node_i;
            js[r] = updates[r].node_j;
            rhos[r] = updates[r].rho;
            any_general |= updates[r].kind == RankOneUpdate::Kind::general;
        }
        if (any_general) {
            vs.assign(k * n, 0.0);
            for (std::size_t r = 0; r < k; ++r)
                if (updates[r].kind == RankOneUpdate::Kind::general) {
                    if (updates[r].v.size() != n)
                        throw std::runtime_error("compose_rank_k: stage " + std::to_string(r + 1) +
                                                 ": RankOneUpdate: direction length mismatch");
                    std::copy(updates[r].v.begin(), updates[r].v.end(), vs.begin() + static_cast<std::ptrdiff_t>(r * n));
                }
        }
        dctp_chain* h = nullptr;
        detail::check(dctp_chain_create(n, k, kinds.data(), is.data(), js.data(), rhos.data(),
                                        any_general ? vs.data() : nullptr, base.path ? nullptr : base.lambda.data(),
                                        base.path ? nullptr : base.u.data(), tau, device, &h));
        h_.reset(h, [](dctp_chain* c) { dctp_chain_destroy(c); });
        mu.resize(n);
        x.resize(n * n);
        detail::check(dctp_chain_spectrum(h, mu.data(), x.data()));
        stages = k;
    }

    std::size_t n = 0, stages = 0;
    std::vector<double> x, mu;

    /// chain_forward for device rows (batch x n), on `stream`.
    void forward_batch(const double* d_in, double* d_out, std::size_t batch, void* stream = nullptr) const {
        detail::check(dctp_chain_forward_f64(h_.get(), d_in, d_out, batch, stream));
    }
    void forward_batch(const float* d_in, float* d_out, std::size_t batch, void* stream = nullptr) const {
        detail::check(dctp_chain_forward_f32(h_.get(), d_in, d_out, batch, stream));
    }
    void sync_check(void* stream = nullptr) const { detail::check(dctp_chain_sync_check(h_.get(), stream)); }
    const dctp_chain* handle() const { return h_.get(); }

  private:
    std::shared_ptr<dctp_chain> h_;
};

inline ChainedFactorization compose_rank_k(const SpectralBasis& base, const std::vector<RankOneUpdate>& updates,
                                           double tau = 1e-12) {
    return ChainedFactorization(base, updates, tau);
}

/// chain_forward (cauchy.hpp:218-231) of one host signal.
inline std::vector<double> chain_forward(const ChainedFactorization& f, const std::vector<double>& s) {
    if (s.size() != f.n) throw std::invalid_argument("chain_forward: size mismatch");
    std::vector<double> out(f.n);
    detail::check(dctp_chain_forward_host_f64(f.handle(), s.data(), out.data(), 1));
    return out;
}

} // namespace dctplus_b200

#endif
