// Per-graph setup of one DCT+ plan, computed once on the host.
//
// This is the product's restatement of DctPlusPlan's constructor
// (proj/include/dctplus/fast_transform.hpp:45-134) and the spectral routines
// it calls (spectral.hpp:30-37, :155-233, :252-315, :340-381; cauchy.hpp:84-103).
// The batched apply consumes mu, the deflated z, the normalisers a and the
// column signs sigma; SURVEY.md section 0.5 shows a 1-ulp change of mu moves
// config-5 outputs by 6.5e-9, so every floating-point operation here is kept
// in the reference's order and the file is compiled with -ffp-contract=off
// (no FMA contraction).  The secular solve, the normalisers and the basis
// columns are independent per root / per column, so they run on a pool of
// host threads without changing a single bit of the result.
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <limits>
#include <numbers>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "host/r2r.hpp"

namespace dctp::host {

/// Rank-one update L + rho v v^T.  self_loop: v = e_i; edge_delta:
/// v = e_i - e_j (graph.hpp:87-114, 1-based vertices).  general: caller's v
/// (the extension config 5 needs).
struct Update {
    enum class Kind : int { self_loop = 0, edge_delta = 1, general = 2 };
    Kind kind = Kind::self_loop;
    double rho = 0.0;
    std::size_t node_i = 0, node_j = 0;
    std::vector<double> v;

    static Update self_loop(std::size_t i, double w) {
        if (i < 1) throw std::invalid_argument("RankOneUpdate: node index is 1-based");
        if (w == 0.0) throw std::invalid_argument("RankOneUpdate: weight must be nonzero");
        return {Kind::self_loop, w, i, 0, {}};
    }
    static Update edge_delta(std::size_t i, std::size_t j, double w) {
        if (i < 1 || i >= j) throw std::invalid_argument("RankOneUpdate: need 1 <= i < j");
        if (w == 0.0) throw std::invalid_argument("RankOneUpdate: weight must be nonzero");
        return {Kind::edge_delta, w, i, j, {}};
    }
    static Update general(std::vector<double> dir, double w) {
        if (dir.empty()) throw std::invalid_argument("RankOneUpdate: empty direction");
        if (w == 0.0) throw std::invalid_argument("RankOneUpdate: weight must be nonzero");
        for (double x : dir)
            if (!std::isfinite(x)) throw std::invalid_argument("RankOneUpdate: non-finite direction");
        return {Kind::general, w, 0, 0, std::move(dir)};
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
};

inline unsigned setup_threads() {
    unsigned t = std::thread::hardware_concurrency();
    return t == 0 ? 1u : t;
}

/// Runs body(i) for i in [0, count) on a small thread pool (dynamic chunks).
inline void parallel_for(std::size_t count, const std::function<void(std::size_t)>& body,
                         std::size_t min_per_thread = 16) {
    const unsigned hw = setup_threads();
    const std::size_t want = std::min<std::size_t>(hw, (count + min_per_thread - 1) / min_per_thread);
    if (want <= 1) {
        for (std::size_t i = 0; i < count; ++i) body(i);
        return;
    }
    std::atomic<std::size_t> next{0};
    std::vector<std::exception_ptr> errs(want);
    std::vector<std::thread> pool;
    for (std::size_t t = 0; t < want; ++t)
        pool.emplace_back([&, t] {
            try {
                for (;;) {
                    const std::size_t i0 = next.fetch_add(8);
                    if (i0 >= count) break;
                    for (std::size_t i = i0; i < std::min(count, i0 + 8); ++i) body(i);
                }
            } catch (...) {
                errs[t] = std::current_exception();
            }
        });
    for (auto& th : pool) th.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

/// Orthonormal DCT-II / its inverse with the reference TrigPlan's rounding:
/// a dense product below length 17 (except length 8), otherwise the r2r core
/// followed by the same scalings (trig.hpp:34-43, :84-116, :131-165).
class Trig {
  public:
    enum class Kind { dct2, idct2 };
    Trig(Kind kind, std::size_t len) : kind_(kind), len_(len) {
        if (len < 1) throw std::invalid_argument("TrigPlan: length must be positive");
        if (len <= 16 && len != 8) {
            const double pi = std::numbers::pi;
            const double nd = static_cast<double>(len);
            dense_.resize(len * len);
            const double scale = std::sqrt(2.0 / nd);
            for (std::size_t k = 0; k < len; ++k) {
                const double ck = (k == 0) ? 1.0 / std::numbers::sqrt2 : 1.0;
                for (std::size_t j = 0; j < len; ++j) {
                    const double u = ck * scale *
                                     std::cos(pi * static_cast<double>(k) *
                                              (2.0 * static_cast<double>(j) + 1.0) / (2.0 * nd));
                    if (kind == Kind::dct2)
                        dense_[k * len + j] = u;
                    else
                        dense_[j * len + k] = u;
                }
            }
            return;
        }
        core_ = r2r::R2r(kind == Kind::dct2 ? r2r::Kind::redft10 : r2r::Kind::redft01, len);
    }

    std::size_t length() const { return len_; }

    /// scratch: at least scratch_size() doubles.
    std::size_t scratch_size() const { return dense_.empty() ? core_.scratch_size() + len_ : 0; }

    void execute(const double* in, double* out, double* scratch) const {
        const std::size_t n = len_;
        if (!dense_.empty()) {
            for (std::size_t i = 0; i < n; ++i) {
                const double* row = dense_.data() + i * n;
                double acc = 0.0;
                for (std::size_t j = 0; j < n; ++j) acc += row[j] * in[j];
                out[i] = acc;
            }
            return;
        }
        const double s = 1.0 / std::sqrt(2.0 * static_cast<double>(n));
        if (kind_ == Kind::dct2) {
            core_.exec(in, out, scratch);
            for (std::size_t i = 0; i < n; ++i) out[i] *= s;
            out[0] *= std::numbers::sqrt2 / 2.0;
        } else {
            double* w = scratch + core_.scratch_size();
            for (std::size_t i = 0; i < n; ++i) w[i] = in[i];
            w[0] *= std::numbers::sqrt2;
            core_.exec(w, out, scratch);
            for (std::size_t i = 0; i < n; ++i) out[i] *= s;
        }
    }

  private:
    Kind kind_;
    std::size_t len_;
    std::vector<double> dense_;
    r2r::R2r core_;
};

// --- secular equation (spectral.hpp:149-233) -----------------------------------

struct SecularValue {
    double f, df, scale;
};

inline SecularValue secular_value(const std::vector<double>& lam, const std::vector<double>& z,
                                  double rho, double x) {
    double sum = 0.0, dsum = 0.0, asum = 0.0;
    const std::size_t m = lam.size();
    for (std::size_t j = 0; j < m; ++j) {
        const double gap = lam[j] - x;
        const double term = z[j] * z[j] / gap;
        sum += term;
        dsum += term / gap;
        asum += std::abs(term);
    }
    return {1.0 + rho * sum, rho * dsum, 1.0 + std::abs(rho) * asum};
}

/// Safeguarded Newton on one interlacing bracket: midpoint start, a forced
/// bisection every fourth step or whenever Newton leaves the bracket.
inline double secular_root(const std::vector<double>& lam, const std::vector<double>& z,
                           double rho, double lo, double hi) {
    const double dir = (rho > 0.0) ? 1.0 : -1.0;
    const double ulp4 = 4.0 * std::numeric_limits<double>::epsilon();
    const double tiny = std::numeric_limits<double>::min();
    double x = 0.5 * (lo + hi);
    for (int it = 0; it < 200; ++it) {
        const SecularValue e = secular_value(lam, z, rho, x);
        if (std::abs(e.f) <= 1e-15 * e.scale) return x;
        if (dir * e.f < 0.0)
            lo = x;
        else
            hi = x;
        if (hi - lo <= ulp4 * (std::abs(lo) + std::abs(hi) + tiny)) return 0.5 * (lo + hi);
        double next = x - e.f / e.df;
        if (!(next > lo && next < hi) || e.df == 0.0 || (it % 4) == 3) next = 0.5 * (lo + hi);
        x = next;
    }
    throw std::runtime_error("secular_eigenvalues: no convergence in 200 iterations");
}

struct Setup;

/// Optional device backend for the two O(k^2) loops of the setup (the GPU
/// kernels in kernels/setup.cu, same operations in the same order, so the
/// results are bit-identical); empty members fall back to the host loops.
struct SecularBackend {
    std::function<std::vector<double>(const std::vector<double>& lam, const std::vector<double>& z, double rho,
                                      double zz)>
        roots;
    std::function<std::vector<double>(const std::vector<double>& lam, const std::vector<double>& mu,
                                      const std::vector<double>& z)>
        normalisers;
    // column signs of the unsigned basis (fills Setup::sigma)
    std::function<void(Setup&)> signs;
};

inline std::vector<double> secular_roots(const std::vector<double>& lam, const std::vector<double>& z,
                                         double rho, const SecularBackend* be = nullptr) {
    const std::size_t k = lam.size();
    if (k == 0) return {};
    if (z.size() != k) throw std::invalid_argument("secular_eigenvalues: size mismatch");
    if (rho == 0.0) throw std::invalid_argument("secular_eigenvalues: rho must be nonzero");
    for (std::size_t j = 0; j < k; ++j) {
        if (z[j] == 0.0)
            throw std::invalid_argument("secular_eigenvalues: zero z component; deflate first");
        if (j + 1 < k && !(lam[j + 1] > lam[j]))
            throw std::invalid_argument("secular_eigenvalues: repeated or unsorted eigenvalues; deflate first");
    }
    double zz = 0.0;
    for (double x : z) zz += x * x;
    std::vector<double> mu(k);
    if (k == 1) {
        mu[0] = lam[0] + rho * zz;
        return mu;
    }
    if (be && be->roots) return be->roots(lam, z, rho, zz);
    // Root r lies in (lo_r, hi_r); the exterior bracket sits on rho's side.
    parallel_for(k, [&](std::size_t r) {
        double lo, hi;
        if (rho > 0.0) {
            lo = lam[r];
            hi = (r + 1 < k) ? lam[r + 1] : lam[k - 1] + rho * zz;
        } else {
            lo = (r == 0) ? lam[0] + rho * zz : lam[r - 1];
            hi = lam[r];
        }
        mu[r] = secular_root(lam, z, rho, lo, hi);
    }, 4);
    return mu;
}

// --- deflation and normalisers (spectral.hpp:242-315) ---------------------------

/// Givens rotation of two base columns: u_into' = c u_into + s u_from,
/// u_from' = -s u_into + c u_from (spectral.hpp:236-250).
struct Rotation {
    std::size_t into, from;
    double c, s;
};

struct Deflated {
    std::vector<std::size_t> kept, passed;
    std::vector<Rotation> rotations;
    std::vector<double> z; // zero at passed indices
};

inline Deflated deflate(const std::vector<double>& lam, const std::vector<double>& z, double tau) {
    if (lam.size() != z.size()) throw std::invalid_argument("deflate: size mismatch");
    if (tau < 0.0) throw std::invalid_argument("deflate: tau must be nonnegative");
    const std::size_t n = lam.size();
    Deflated d;
    d.z = z;
    double lmax = 0.0;
    for (double x : lam) lmax = std::max(lmax, std::abs(x));
    const double gap_tol = tau * lmax;
    // Near-equal eigenvalue runs fold their z mass onto the run's first entry.
    std::size_t first = 0;
    for (std::size_t j = 1; j <= n; ++j) {
        if (j < n && lam[j] - lam[j - 1] <= gap_tol) continue;
        for (std::size_t k = first + 1; k < j; ++k) {
            const double zf = d.z[first], zk = d.z[k];
            const double h = std::hypot(zf, zk);
            if (h > 0.0) {
                d.rotations.push_back({first, k, zf / h, zk / h});
                d.z[first] = h;
            }
            d.z[k] = 0.0;
        }
        first = j;
    }
    double znorm = 0.0;
    for (double x : d.z) znorm = std::hypot(znorm, x);
    const double z_tol = tau * znorm;
    for (std::size_t j = 0; j < n; ++j) {
        if (std::abs(d.z[j]) <= z_tol) {
            d.z[j] = 0.0;
            d.passed.push_back(j);
        } else {
            d.kept.push_back(j);
        }
    }
    return d;
}

inline std::vector<double> normalisers(const std::vector<double>& lam, const std::vector<double>& mu,
                                       const std::vector<double>& z, const SecularBackend* be = nullptr) {
    if (lam.size() != z.size()) throw std::invalid_argument("normalizers: size mismatch");
    if (be && be->normalisers) return be->normalisers(lam, mu, z);
    std::vector<double> a(mu.size());
    std::vector<int> bad(mu.size(), 0);
    parallel_for(mu.size(), [&](std::size_t i) {
        double s = 0.0;
        for (std::size_t j = 0; j < lam.size(); ++j) {
            const double d = mu[i] - lam[j];
            if (d == 0.0 && z[j] != 0.0) {
                bad[i] = 1;
                return;
            }
            if (z[j] != 0.0) s += (z[j] / d) * (z[j] / d);
        }
        if (!(s > 0.0) || !std::isfinite(s)) {
            bad[i] = 2;
            return;
        }
        a[i] = 1.0 / std::sqrt(s);
    }, 4);
    for (int b : bad) {
        if (b == 1) throw std::domain_error("normalizers: mu/lambda collision; deflation missing");
        if (b == 2) throw std::domain_error("normalizers: degenerate column");
    }
    return a;
}

/// sign making the largest-magnitude entry positive; ties within 1e-12
/// relative go to the lowest row (spectral.hpp:30-37).
inline double sign_of_column(const double* col, std::size_t n) {
    double peak = 0.0;
    for (std::size_t i = 0; i < n; ++i) peak = std::max(peak, std::abs(col[i]));
    if (peak == 0.0) return 1.0;
    for (std::size_t i = 0; i < n; ++i)
        if (std::abs(col[i]) >= peak * (1.0 - 1e-12)) return col[i] < 0.0 ? -1.0 : 1.0;
    return 1.0;
}

// --- perturbed spectrum (spectral.hpp:318-381) -----------------------------------

struct Slot {
    bool passthrough;
    std::size_t idx; // passthrough: DCT index; active: rank in the secular subproblem
};

/// perturb_spectrum (spectral.hpp:340-381): deflate, solve the secular
/// subproblem, and merge pass-through eigenvalues with the roots into one
/// ascending list of slots.
struct Perturbed {
    std::vector<double> z, mu, a; // z deflated; a per slot (1 for pass-through)
    std::vector<Slot> slots;
    std::vector<Rotation> rotations;
    std::vector<std::size_t> kept, passed;
    std::vector<double> sub_lambda, sub_z, sub_mu;
};

inline Perturbed perturb_spectrum(const std::vector<double>& lam, const std::vector<double>& z, double rho,
                                  double tau, const SecularBackend* be = nullptr) {
    Perturbed p;
    Deflated d = deflate(lam, z, tau);
    p.z = std::move(d.z);
    p.kept = std::move(d.kept);
    p.passed = std::move(d.passed);
    p.rotations = std::move(d.rotations);
    for (std::size_t j : p.kept) {
        p.sub_lambda.push_back(lam[j]);
        p.sub_z.push_back(p.z[j]);
    }
    if (!p.sub_lambda.empty()) p.sub_mu = secular_roots(p.sub_lambda, p.sub_z, rho, be);
    const std::vector<double> sub_a =
        p.sub_mu.empty() ? std::vector<double>{} : normalisers(p.sub_lambda, p.sub_mu, p.sub_z, be);

    std::size_t ip = 0, ia = 0;
    const std::size_t n = lam.size();
    p.mu.reserve(n);
    p.slots.reserve(n);
    p.a.reserve(n);
    while (ip < p.passed.size() || ia < p.sub_mu.size()) {
        const bool pass_first =
            ia == p.sub_mu.size() || (ip < p.passed.size() && lam[p.passed[ip]] <= p.sub_mu[ia]);
        if (pass_first) {
            p.mu.push_back(lam[p.passed[ip]]);
            p.slots.push_back({true, p.passed[ip]});
            p.a.push_back(1.0);
            ++ip;
        } else {
            p.mu.push_back(p.sub_mu[ia]);
            p.slots.push_back({false, ia});
            p.a.push_back(sub_a[ia]);
            ++ia;
        }
    }
    return p;
}

// --- the assembled setup (fast_transform.hpp:45-134) -----------------------------

struct Setup {
    std::size_t n = 0;
    double rho = 0.0, epsilon = 0.0, tau = 0.0;
    std::vector<double> lambda, z_raw, z, mu, a, sigma;
    std::vector<Slot> slots;
    std::vector<std::size_t> kept, passed;
    std::vector<double> sub_mu;
    bool slow_path = false;
};

/// y-vector of column `s` of the unsigned basis in the DCT domain
/// (cauchy.hpp:90-98): pass-through e_idx, active a_s z_j / (lambda_j - nu).
inline void basis_coefficients(const Setup& st, std::size_t s, double* y) {
    const std::size_t n = st.n;
    std::fill(y, y + n, 0.0);
    if (st.slots[s].passthrough) {
        y[st.slots[s].idx] = 1.0;
        return;
    }
    const double nu = st.sub_mu[st.slots[s].idx];
    for (std::size_t j = 0; j < n; ++j)
        if (st.z[j] != 0.0) y[j] = st.a[s] * st.z[j] / (st.lambda[j] - nu);
}

inline Setup build_setup(std::size_t n, const Update& update, double epsilon, double tau,
                         const SecularBackend* be = nullptr) {
    if (n < 2) throw std::invalid_argument("DctPlusPlan: need n >= 2");
    if (!(epsilon > 0.0) || !(epsilon < 1.0))
        throw std::invalid_argument("DctPlusPlan: epsilon must lie in (0, 1)");
    Setup st;
    st.n = n;
    st.rho = update.rho;
    st.epsilon = epsilon;
    st.tau = tau;

    const double pi = std::numbers::pi;
    st.lambda.resize(n);
    for (std::size_t k = 0; k < n; ++k)
        st.lambda[k] = 2.0 - 2.0 * std::cos(static_cast<double>(k) * pi / static_cast<double>(n));
    st.lambda[0] = 0.0;

    const std::vector<double> v = update.direction(n);
    const Trig dct(Trig::Kind::dct2, n);
    st.z_raw.resize(n);
    {
        std::vector<double> scratch(dct.scratch_size() + 1);
        dct.execute(v.data(), st.z_raw.data(), scratch.data());
    }

    Perturbed ps = perturb_spectrum(st.lambda, st.z_raw, update.rho, tau, be);
    if (!ps.rotations.empty()) throw std::logic_error("DctPlusPlan: path eigenvalues cannot repeat");
    st.z = std::move(ps.z);
    st.kept = std::move(ps.kept);
    st.passed = std::move(ps.passed);
    st.sub_mu = std::move(ps.sub_mu);
    st.mu = std::move(ps.mu);
    st.slots = std::move(ps.slots);
    st.a = std::move(ps.a);

    // Column signs from the materialised basis, one inverse DCT per column
    // (cauchy.hpp:84-103 through fast_transform.hpp:72-84).
    st.sigma.assign(n, 1.0);
    if (be && be->signs) {
        be->signs(st);
    } else {
    const Trig idct(Trig::Kind::idct2, n);
    parallel_for(n, [&](std::size_t s) {
        thread_local std::vector<double> buf;
        const std::size_t need = 2 * n + idct.scratch_size() + 1;
        if (buf.size() < need) buf.resize(need);
        double* y = buf.data();
        double* col = y + n;
        basis_coefficients(st, s, y);
        idct.execute(y, col, col + n);
        st.sigma[s] = sign_of_column(col, n);
    }, 4);
    }

    // slow_path() exactly as the reference decides it (fast_transform.hpp:86-117):
    // a near-pole secular root, or an interior root outside the Chebyshev range.
    const double guard = 1e-10 * st.lambda[n - 1];
    for (double nu : st.sub_mu)
        for (double l : st.lambda)
            if (std::abs(nu - l) < guard) st.slow_path = true;
    if (!st.slow_path) {
        const std::size_t na = st.sub_mu.size();
        const std::size_t ext_rank = (na == 0) ? 0 : (update.rho > 0.0 ? na - 1 : 0);
        for (const Slot& sl : st.slots) {
            if (sl.passthrough || (na > 0 && sl.idx == ext_rank)) continue;
            const double mu_t = 1.0 - st.sub_mu[sl.idx] / 2.0;
            if (!(mu_t > -1.0 && mu_t < 1.0)) {
                st.slow_path = true;
                break;
            }
        }
    }
    return st;
}

} // namespace dctp::host
