// ORACLE TEST INFRASTRUCTURE — never linked into the product.
//
// C-ABI driver over the UNMODIFIED reference headers under
// /root/reference/proj/include (plus the general-direction patch of graph.hpp
// that oracle/build_ref.sh writes into oracle/_ref/include),
// compiled against the FFTW stand-in in oracle/fftw_shim.  Built into
// oracle/_ref/libdctref.so; used by tests/ (goldens, parity), by
// oracle/gen_golden.py and by bench.py's CPU-baseline / --impl reference leg.
//
// Threading follows the reference's documented model (proj/README.md:82-87,
// fast_transform.hpp:33-34): one shared immutable plan, one workspace per
// std::thread, each thread owning a contiguous slice of the batch.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "dctplus/dctplus.hpp"

using namespace dctplus;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
    if (dynamic_cast<const std::domain_error*>(&e)) return 2;
    if (dynamic_cast<const std::logic_error*>(&e)) return 4;
    return 3;
}

RankOneUpdate make_update(int kind, std::size_t i, std::size_t j, double rho, const double* v,
                          std::size_t n) {
    if (kind == 0) return RankOneUpdate::self_loop(i, rho);
    if (kind == 1) return RankOneUpdate::edge_delta(i, j, rho);
    if (kind == 2) {
        if (rho == 0.0) throw std::invalid_argument("RankOneUpdate: weight must be nonzero");
        RankOneUpdate u{RankOneUpdate::Kind::self_loop, rho, 0, 0};
        u.general_v.assign(v, v + n);
        return u;
    }
    throw std::invalid_argument("ref_driver: unknown update kind");
}

template <class F>
void parallel_slices(std::size_t batch, int threads, F&& body) {
    if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    threads = static_cast<int>(std::min<std::size_t>(static_cast<std::size_t>(threads), std::max<std::size_t>(batch, 1)));
    if (threads <= 1) {
        body(std::size_t{0}, batch);
        return;
    }
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errs(static_cast<std::size_t>(threads));
    const std::size_t per = (batch + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const std::size_t b0 = std::min(batch, per * t), b1 = std::min(batch, per * (t + 1));
        pool.emplace_back([&, t, b0, b1] {
            try {
                body(b0, b1);
            } catch (...) {
                errs[static_cast<std::size_t>(t)] = std::current_exception();
            }
        });
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_plan_create(std::size_t n, int kind, std::size_t i, std::size_t j, double rho,
                    const double* v, double eps, double tau, void** out) {
    try {
        *out = new DctPlusPlan(n, make_update(kind, i, j, rho, v, n), eps, tau);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void ref_plan_destroy(void* p) { delete static_cast<DctPlusPlan*>(p); }

int ref_plan_slow_path(const void* p) { return static_cast<const DctPlusPlan*>(p)->slow_path() ? 1 : 0; }

/// Setup vectors: lambda, deflated z, mu, a (per slot), sigma (per slot),
/// slot_pass / slot_idx (SlotRef), sub_mu (na entries); counts via n_sub.
int ref_plan_setup(const void* pv, double* lambda, double* z, double* mu, double* a,
                   double* sigma, int* slot_pass, std::int64_t* slot_idx, double* sub_mu,
                   std::size_t* n_sub) {
    const auto* p = static_cast<const DctPlusPlan*>(pv);
    const auto& f = p->factorization();
    const std::size_t n = p->size();
    for (std::size_t k = 0; k < n; ++k) {
        if (lambda) lambda[k] = p->lambda()[k];
        if (z) z[k] = f.spec.z[k];
        if (mu) mu[k] = f.spec.mu[k];
        if (a) a[k] = f.spec.a[k];
        if (sigma) sigma[k] = f.sigma[k];
        if (slot_pass) slot_pass[k] = f.spec.slots[k].passthrough ? 1 : 0;
        if (slot_idx) slot_idx[k] = static_cast<std::int64_t>(f.spec.slots[k].idx);
    }
    if (sub_mu)
        for (std::size_t k = 0; k < f.spec.sub_mu.size(); ++k) sub_mu[k] = f.spec.sub_mu[k];
    if (n_sub) *n_sub = f.spec.sub_mu.size();
    return 0;
}

/// Batched DctPlusPlan::forward (fast_transform.hpp:163-190); mode 1 runs
/// forward_nmvp (:199-209) instead.
int ref_forward(const void* pv, const double* s, double* out, std::size_t batch, int mode,
                int threads) {
    try {
        const auto* p = static_cast<const DctPlusPlan*>(pv);
        const std::size_t n = p->size();
        parallel_slices(batch, threads, [&](std::size_t b0, std::size_t b1) {
            DctPlusWorkspace ws = p->make_workspace();
            std::vector<double> sig(n);
            for (std::size_t b = b0; b < b1; ++b) {
                std::copy(s + b * n, s + (b + 1) * n, sig.begin());
                const std::vector<double>& r =
                    (mode == 1) ? p->forward_nmvp(sig, ws) : p->forward(sig, ws);
                std::copy(r.begin(), r.end(), out + b * n);
            }
        });
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/// Batched DctPlusPlan::inverse (fast_transform.hpp:218-255).
int ref_inverse(const void* pv, const double* pin, double* out, std::size_t batch, int fast,
                int threads) {
    try {
        const auto* p = static_cast<const DctPlusPlan*>(pv);
        const std::size_t n = p->size();
        parallel_slices(batch, threads, [&](std::size_t b0, std::size_t b1) {
            DctPlusWorkspace ws = p->make_workspace();
            std::vector<double> sig(n);
            for (std::size_t b = b0; b < b1; ++b) {
                std::copy(pin + b * n, pin + (b + 1) * n, sig.begin());
                const std::vector<double>& r = p->inverse(sig, ws, fast != 0);
                std::copy(r.begin(), r.end(), out + b * n);
            }
        });
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_ensemble_create(std::size_t n, std::size_t k, const int* kinds, const std::size_t* is,
                        const std::size_t* js, const double* rhos, const double* vs,
                        std::size_t cp, double threshold, double eps, void** out) {
    try {
        std::vector<RankOneUpdate> ups;
        for (std::size_t r = 0; r < k; ++r)
            ups.push_back(make_update(kinds[r], is[r], js[r], rhos[r], vs ? vs + r * n : nullptr, n));
        *out = new PrunedEnsemblePlan(n, ups, cp, threshold, eps);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void ref_ensemble_destroy(void* p) { delete static_cast<PrunedEnsemblePlan*>(p); }

const void* ref_ensemble_member(const void* p, std::size_t r) {
    return &static_cast<const PrunedEnsemblePlan*>(p)->member(r);
}

/// Batched PrunedEnsemblePlan::forward_all (fast_transform.hpp:396-439);
/// out is [batch][K+1][n], set 0 = the shared DCT; pruned flags per signal.
int ref_ensemble_forward_all(const void* pv, const double* s, double* out, int* pruned,
                             std::size_t batch, int threads) {
    try {
        const auto* p = static_cast<const PrunedEnsemblePlan*>(pv);
        const std::size_t n = p->size(), sets = p->ensemble_size();
        parallel_slices(batch, threads, [&](std::size_t b0, std::size_t b1) {
            PrunedWorkspace ws = p->make_workspace();
            PrunedEnsemblePlan::Result res;
            std::vector<double> sig(n);
            for (std::size_t b = b0; b < b1; ++b) {
                std::copy(s + b * n, s + (b + 1) * n, sig.begin());
                p->forward_all(sig, ws, res);
                for (std::size_t r = 0; r < sets; ++r)
                    std::copy(res.coeffs[r].begin(), res.coeffs[r].end(), out + (b * sets + r) * n);
                if (pruned) pruned[b] = res.pruned ? 1 : 0;
            }
        });
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/// forward_all with bounds: bounds is [batch][K+1] (Result::bounds).
int ref_ensemble_forward_all_bounds(const void* pv, const double* s, double* out, double* bounds, int* pruned,
                                    std::size_t batch, int threads) {
    try {
        const auto* p = static_cast<const PrunedEnsemblePlan*>(pv);
        const std::size_t n = p->size(), sets = p->ensemble_size();
        parallel_slices(batch, threads, [&](std::size_t b0, std::size_t b1) {
            PrunedWorkspace ws = p->make_workspace();
            PrunedEnsemblePlan::Result res;
            std::vector<double> sig(n);
            for (std::size_t b = b0; b < b1; ++b) {
                std::copy(s + b * n, s + (b + 1) * n, sig.begin());
                p->forward_all(sig, ws, res);
                for (std::size_t r = 0; r < sets; ++r) {
                    std::copy(res.coeffs[r].begin(), res.coeffs[r].end(), out + (b * sets + r) * n);
                    bounds[b * sets + r] = res.bounds[r];
                }
                pruned[b] = res.pruned ? 1 : 0;
            }
        });
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/// rdo_select (fast_transform.hpp:494-496, l1 cost) per signal: index, pruned.
int ref_rdo_select(const void* pv, const double* s, int* index, int* pruned, std::size_t batch) {
    try {
        const auto* p = static_cast<const PrunedEnsemblePlan*>(pv);
        const std::size_t n = p->size();
        for (std::size_t b = 0; b < batch; ++b) {
            const std::vector<double> sig(s + b * n, s + (b + 1) * n);
            const RdoChoice c = rdo_select(*p, sig);
            index[b] = static_cast<int>(c.index);
            pruned[b] = c.pruned ? 1 : 0;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/// compose_rank_k (cauchy.hpp:175-216) on path_spectrum(n) (base NULL) or a
/// caller's base (lambda n, u n x n row-major).
int ref_chain_create(std::size_t n, std::size_t k, const int* kinds, const std::size_t* is, const std::size_t* js,
                     const double* rhos, const double* vs, const double* base_lambda, const double* base_u,
                     double tau, void** out) {
    try {
        std::vector<RankOneUpdate> ups;
        for (std::size_t r = 0; r < k; ++r)
            ups.push_back(make_update(kinds[r], is[r], js[r], rhos[r], vs ? vs + r * n : nullptr, n));
        SpectralBasis base;
        if (base_lambda) {
            base.lambda.assign(base_lambda, base_lambda + n);
            base.u = Matrix(n, n);
            for (std::size_t i = 0; i < n; ++i)
                for (std::size_t j = 0; j < n; ++j) base.u(i, j) = base_u[i * n + j];
        } else {
            base = path_spectrum(n);
        }
        *out = new ChainedFactorization(compose_rank_k(base, ups, tau));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void ref_chain_destroy(void* p) { delete static_cast<ChainedFactorization*>(p); }

/// ChainedFactorization::mu, ::x (row-major), stage count.
int ref_chain_spectrum(const void* pv, double* mu, double* x, std::size_t* stages) {
    const auto* c = static_cast<const ChainedFactorization*>(pv);
    const std::size_t n = c->n;
    for (std::size_t i = 0; i < n; ++i) {
        mu[i] = c->mu[i];
        for (std::size_t j = 0; j < n; ++j) x[i * n + j] = c->x(i, j);
    }
    *stages = c->stages.size();
    return 0;
}

/// chain_forward (cauchy.hpp:218-231) per signal.
int ref_chain_forward(const void* pv, const double* s, double* out, std::size_t batch, int threads) {
    try {
        const auto* c = static_cast<const ChainedFactorization*>(pv);
        const std::size_t n = c->n;
        parallel_slices(batch, threads, [&](std::size_t b0, std::size_t b1) {
            for (std::size_t b = b0; b < b1; ++b) {
                const std::vector<double> sig(s + b * n, s + (b + 1) * n);
                const std::vector<double> p = chain_forward(*c, sig);
                std::copy(p.begin(), p.end(), out + b * n);
            }
        });
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/// bench.hpp:26-64: parse_update + format_update of a descriptor (1 on a bad
/// one, message in ref_last_error) and one csv_row.
int ref_format_update(const char* text, char* out, std::size_t len) {
    try {
        const std::string s = format_update(parse_update(text));
        std::snprintf(out, len, "%s", s.c_str());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void ref_csv_row(const char* mode, std::size_t size, const char* update, const char* method, const char* metric,
                 double value, char* out, std::size_t len) {
    std::ostringstream os;
    csv_row(os, mode, size, update, method, metric, value);
    std::snprintf(out, len, "%s", os.str().c_str());
}

/// bench.hpp:99-108.
double ref_calibrate_prune_threshold(std::size_t n, double r, double quantile, std::size_t trials,
                                     std::uint64_t seed) {
    return calibrate_prune_threshold(n, r, quantile, trials, seed);
}

/// trig.hpp TrigPlan execute (kind 0 dct2, 1 idct2, 2 dst1) on `count` rows.
int ref_trig(int kind, std::size_t len, const double* in, double* out, std::size_t count) {
    try {
        TrigPlan plan(kind == 0 ? TrigKind::dct2 : (kind == 1 ? TrigKind::idct2 : TrigKind::dst1), len);
        std::vector<double> work(len);
        for (std::size_t b = 0; b < count; ++b) plan.execute(in + b * len, out + b * len, work.data());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// --- signal.hpp / bench.hpp harness --------------------------------------------

std::uint64_t ref_mix_seed(std::uint64_t seed, std::size_t size, std::size_t kind) {
    return mix_seed(seed, size, kind);
}

/// dist 0: gaussian(), 1: uniform(), 2: rows of gen_ar_signal(n, r).
void ref_rng_fill(std::uint64_t seed, int dist, double r, std::size_t n, std::size_t rows,
                  double* out) {
    Rng rng(seed);
    if (dist == 2) {
        for (std::size_t b = 0; b < rows; ++b) {
            const auto s = gen_ar_signal(n, r, rng);
            std::copy(s.begin(), s.end(), out + b * n);
        }
        return;
    }
    for (std::size_t i = 0; i < n * rows; ++i) out[i] = dist == 0 ? rng.gaussian() : rng.uniform();
}

} // extern "C"
