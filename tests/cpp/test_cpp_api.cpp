// C++ mirror API test (include/dctplus_b200/dctplus.hpp), written like the
// reference's own suites (proj/tests/test_fast_transform.cpp,
// test_spectral.cpp, test_pruning.cpp): known answers, dense-oracle checks,
// SNR >= 100 dB, exception classes.  Prints "ALL OK" and exits 0 on success.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <cstdlib>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime_api.h>

#include "dctplus_b200/dctplus.hpp"

namespace dctplus = dctplus_b200;
using namespace dctplus;

static int failures = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        if (!(cond)) {                                                         \
            std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
            ++failures;                                                        \
        }                                                                      \
    } while (0)
template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static double snr_db(const std::vector<double>& ref, const std::vector<double>& t) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < ref.size(); ++i) {
        num += ref[i] * ref[i];
        den += (ref[i] - t[i]) * (ref[i] - t[i]);
    }
    return den == 0 ? 320.0 : 10 * std::log10(num / den);
}

static std::vector<double> ar(std::size_t n, double r, std::mt19937_64& g) {
    std::normal_distribution<double> nd;
    std::vector<double> s(n);
    s[0] = nd(g) / std::sqrt(1 - r * r);
    for (std::size_t j = 1; j < n; ++j) s[j] = r * s[j - 1] + nd(g);
    return s;
}

int main() {
    // test_spectral.cpp:129-135 / test_cauchy.cpp:91-100: n = 2 self-loop
    {
        const DctPlusPlan plan(2, RankOneUpdate::self_loop(1, 1.0), 1e-12);
        const auto mu = plan.mu();
        CHECK(std::abs(mu[0] - (3 - std::sqrt(5.0)) / 2) < 1e-14);
        CHECK(std::abs(mu[1] - (3 + std::sqrt(5.0)) / 2) < 1e-14);
    }
    // test_fast_transform.cpp:19-44: interleaving on the three update types
    const std::vector<RankOneUpdate> kBench = {RankOneUpdate::self_loop(1, 1.5), RankOneUpdate::edge_delta(2, 3, 1.5),
                                               RankOneUpdate::edge_delta(3, 5, 1.5)};
    for (const auto& u : kBench) {
        const DctPlusPlan plan(8, u, 1e-12);
        CHECK(!plan.slow_path());
        const auto lam = plan.lambda(), mu = plan.mu();
        for (std::size_t i = 0; i < 8; ++i) {
            CHECK(mu[i] >= lam[i]);
            if (i + 1 < 8) CHECK(mu[i] <= lam[i + 1]);
        }
    }
    // forward vs the dense basis (X^T s) and SNR >= 100 dB round trip
    std::mt19937_64 g(101);
    for (std::size_t n : {8, 32, 128, 256}) {
        for (const auto& u : kBench) {
            const DctPlusPlan plan(n, u, 1e-12);
            const auto x = plan.basis();
            DctPlusWorkspace ws = plan.make_workspace();
            for (int rep = 0; rep < 4; ++rep) {
                const auto s = ar(n, 0.99, g);
                const std::vector<double> fast = plan.forward(s, ws);
                std::vector<double> dense(n, 0.0);
                for (std::size_t i = 0; i < n; ++i)
                    for (std::size_t j = 0; j < n; ++j) dense[j] += x(i, j) * s[i];
                CHECK(snr_db(dense, fast) >= 100.0);
                const auto back = plan.inverse(fast);
                CHECK(snr_db(s, back) >= 100.0);
            }
        }
    }
    // errors (fast_transform.hpp:52-53, :266-276)
    CHECK(throws<std::invalid_argument>([] { DctPlusPlan(1, RankOneUpdate::self_loop(1, 1.0), 1e-12); }));
    CHECK(throws<std::invalid_argument>([] { DctPlusPlan(8, RankOneUpdate::self_loop(1, 1.0), 2.0); }));
    CHECK(throws<std::invalid_argument>([] { RankOneUpdate::edge_delta(3, 3, 1.0); }));
    {
        const DctPlusPlan plan(16, RankOneUpdate::self_loop(1, 0.5), 1e-12);
        std::vector<double> bad(16, 0.0);
        bad[3] = std::nan("");
        CHECK(throws<std::domain_error>([&] { plan.forward(bad); }));
        CHECK(throws<std::invalid_argument>([&] { plan.forward(std::vector<double>(15, 0.0)); }));
    }
    // progressive mode (test_pruning.cpp:35-48): members reproduce the full transforms
    {
        std::vector<RankOneUpdate> ups;
        for (int k = 0; k < 4; ++k) ups.push_back(RankOneUpdate::self_loop(1, 0.05 + 0.5 * k));
        const PrunedEnsemblePlan ens(64, ups, 64, 1e300);
        CHECK(ens.ensemble_size() == 5);
        const auto s = ar(64, 0.9, g);
        const auto res = ens.forward_all(s);
        CHECK(res.pruned);
        for (std::size_t r = 1; r <= 4; ++r) CHECK(snr_db(ens.member(r).forward(s), res.coeffs[r]) >= 100.0);
        CHECK(throws<std::logic_error>([&] { ens.member(0); }));
        CHECK(rdo_select(ens, std::vector<double>(64, 1.0)).index == 0); // test_pruning.cpp:136-141
    }
    // pruned mode (test_pruning.cpp:95-115): the truncation error never exceeds the bound
    {
        const std::vector<RankOneUpdate> ups = {RankOneUpdate::self_loop(1, 1.5), RankOneUpdate::edge_delta(2, 3, 1.5)};
        const PrunedEnsemblePlan ens(32, ups, 16, 1e300);
        for (int rep = 0; rep < 10; ++rep) {
            const auto s = ar(32, 0.99, g);
            const auto res = ens.forward_all(s);
            CHECK(res.pruned);
            for (std::size_t r = 1; r < ens.ensemble_size(); ++r) {
                const auto exact = ens.member(r).forward_nmvp(s); // dense X^T s on the GPU
                double err = 0.0;
                for (std::size_t j = 0; j < 32; ++j) err += (exact[j] - res.coeffs[r][j]) * (exact[j] - res.coeffs[r][j]);
                CHECK(std::sqrt(err) <= res.bounds[r] + 1e-12);
            }
        }
        CHECK(calibrate_prune_threshold(32) > 0.0);
    }
    // batched device rows
    {
        const std::size_t n = 256, batch = 1000;
        const DctPlusPlan plan(n, RankOneUpdate::edge_delta(128, 129, -0.7), 1e-12);
        std::vector<double> h(n * batch), y(n * batch);
        for (std::size_t b = 0; b < batch; ++b) {
            const auto s = ar(n, 0.95, g);
            std::copy(s.begin(), s.end(), h.begin() + static_cast<std::ptrdiff_t>(b * n));
        }
        double *din = nullptr, *dout = nullptr;
        cudaMalloc(reinterpret_cast<void**>(&din), h.size() * 8);
        cudaMalloc(reinterpret_cast<void**>(&dout), h.size() * 8);
        cudaMemcpy(din, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        plan.forward_batch(din, dout, batch);
        plan.sync_check();
        cudaMemcpy(y.data(), dout, y.size() * 8, cudaMemcpyDeviceToHost);
        for (std::size_t b = 0; b < batch; b += 97) {
            const std::vector<double> s(h.begin() + static_cast<std::ptrdiff_t>(b * n),
                                        h.begin() + static_cast<std::ptrdiff_t>((b + 1) * n));
            const std::vector<double> yb(y.begin() + static_cast<std::ptrdiff_t>(b * n),
                                         y.begin() + static_cast<std::ptrdiff_t>((b + 1) * n));
            CHECK(snr_db(plan.forward(s), yb) >= 200.0);
        }
        cudaFree(din);
        cudaFree(dout);
    }
    // rank-k chains (test_cauchy.cpp:203-255): the chain agrees with its own
    // basis, a cancelling pair restores the base spectrum, errors name the stage
    {
        const std::size_t n = 8;
        const auto base = path_spectrum(n);
        const auto chain = compose_rank_k(base, {RankOneUpdate::self_loop(1, 1.5), RankOneUpdate::self_loop(n, 0.8)});
        CHECK(chain.stages == 2);
        const auto s = ar(n, 0.9, g);
        const auto got = chain_forward(chain, s);
        std::vector<double> dense(n, 0.0);
        for (std::size_t i = 0; i < n; ++i)
            for (std::size_t k = 0; k < n; ++k) dense[k] += chain.x[i * n + k] * s[i];
        CHECK(snr_db(dense, got) >= 200.0);
        const auto cancel =
            compose_rank_k(base, {RankOneUpdate::self_loop(2, 0.9), RankOneUpdate::self_loop(2, -0.9)});
        for (std::size_t k = 0; k < n; ++k) CHECK(std::abs(cancel.mu[k] - base.lambda[k]) < 1e-8);
        CHECK(throws<std::invalid_argument>([&] { compose_rank_k(path_spectrum(4), {}); }));
        bool named = false;
        try {
            compose_rank_k(base, {RankOneUpdate::self_loop(1, 1.5), RankOneUpdate::self_loop(99, 1.0)});
        } catch (const std::runtime_error& e) {
            named = std::string(e.what()).find("stage 2") != std::string::npos;
        }
        CHECK(named);
    }
    // test_pruning.cpp:22-48 with the workspace overload (fast_transform.hpp:389-439)
    {
        const std::vector<RankOneUpdate> kEnsembleUpdates = {RankOneUpdate::self_loop(1, 1.5),
                                                             RankOneUpdate::edge_delta(2, 3, 1.5)};
        const double kAlwaysPrune = std::numeric_limits<double>::max();
        CHECK(throws<std::invalid_argument>([&] { PrunedEnsemblePlan(16, kEnsembleUpdates, 0, 1.0); }));
        CHECK(throws<std::invalid_argument>([&] { PrunedEnsemblePlan(16, kEnsembleUpdates, 17, 1.0); }));
        {   // k = 1 degenerates to the plain DCT
            const PrunedEnsemblePlan plan(16, {}, 16, kAlwaysPrune);
            CHECK(plan.ensemble_size() == 1);
            std::vector<double> s(16);
            detail::check(dctp_fill_signals(7, 2, 0.99, 16, 1, s.data()));
            const auto res = plan.forward_all(s);
            CHECK(res.coeffs.size() == 1);
            const TrigPlan dct(TrigKind::dct2, 16);
            const auto d = dct(s);
            double diff = 0.0;
            for (std::size_t j = 0; j < 16; ++j) diff = std::max(diff, std::abs(d[j] - res.coeffs[0][j]));
            CHECK(diff < 1e-14);
        }
        {   // c_p = n reproduces the full transforms; Rng(11), five AR(0.99) signals
            const std::size_t n = 16;
            const PrunedEnsemblePlan plan(n, kEnsembleUpdates, n, kAlwaysPrune);
            std::vector<double> sig(5 * n);
            detail::check(dctp_fill_signals(11, 2, 0.99, n, 5, sig.data()));
            PrunedWorkspace ws = plan.make_workspace();
            PrunedEnsemblePlan::Result res;
            for (int rep = 0; rep < 5; ++rep) {
                const std::vector<double> s(sig.begin() + rep * n, sig.begin() + (rep + 1) * n);
                plan.forward_all(s, ws, res);
                CHECK(res.pruned);
                CHECK(res.coeffs.size() == plan.ensemble_size());
                for (std::size_t r = 1; r < plan.ensemble_size(); ++r)
                    CHECK(snr_db(plan.member(r).forward(s), res.coeffs[r]) >= 100.0);
            }
        }
        {   // accessors by const reference (fast_transform.hpp:136-143, 262)
            const DctPlusPlan plan(64, RankOneUpdate::edge_delta(10, 40, 0.7), 1e-12);
            const CauchyFactorization& f = plan.factorization();
            CHECK(&plan.mu() == &f.mu());
            CHECK(&plan.lambda() == &f.lambda);
            CHECK(f.size() == 64 && f.rho() == 0.7);
            CHECK(f.spec.slots.size() == 64 && f.sigma.size() == 64);
            std::size_t active = 0;
            for (const auto& sl : f.spec.slots) active += sl.passthrough ? 0 : 1;
            CHECK(active == f.spec.sub_mu.size() && f.spec.sub_lambda.size() == f.spec.sub_z.size());
            CHECK(&plan.basis() == &plan.basis() && plan.basis().rows() == 64);
            CHECK(plan.dct_plan().size() == 64);
        }
    }
    // the reference's threading contract (fast_transform.hpp:33-34, README.md:82-87): one
    // shared plan, four host threads on their own streams; a NaN in thread 2's batch raises
    // std::domain_error in thread 2's call only (per-stream flags)
    {
        const std::size_t n = 256, batch = 512;
        const DctPlusPlan plan(n, RankOneUpdate::edge_delta(128, 129, -0.7), 1e-12);
        std::vector<double> h(n * batch);
        detail::check(dctp_fill_signals(5, 2, 0.95, n, batch, h.data()));
        for (int use_per_thread_stream = 0; use_per_thread_stream < 2; ++use_per_thread_stream) {
            int outcome[4] = {0, 0, 0, 0}; // 1 ok, 2 domain_error, 3 other
            std::vector<std::thread> pool;
            for (int t = 0; t < 4; ++t)
                pool.emplace_back([&, t] {
                    cudaStream_t st = cudaStreamPerThread;
                    if (!use_per_thread_stream) cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
                    double *din = nullptr, *dout = nullptr;
                    cudaMalloc(reinterpret_cast<void**>(&din), n * batch * 8);
                    cudaMalloc(reinterpret_cast<void**>(&dout), n * batch * 8);
                    std::vector<double> mine = h;
                    if (t == 2) mine[77 * n + 5] = std::nan("");
                    // on the thread's own stream: a pageable cudaMemcpy may return before its DMA
                    // lands, and a non-blocking stream does not order behind the legacy stream
                    cudaMemcpyAsync(din, mine.data(), n * batch * 8, cudaMemcpyHostToDevice, st);
                    int res = 1;
                    for (int it = 0; it < 20 && res == 1; ++it) {
                        try {
                            plan.forward_batch(din, dout, batch, st);
                            plan.sync_check(st);
                        } catch (const std::domain_error&) {
                            res = 2;
                        } catch (...) {
                            res = 3;
                        }
                    }
                    // the host-buffer path of the same thread: isolated too
                    try {
                        std::vector<double> y(n * batch);
                        plan.forward_host(mine.data(), y.data(), batch);
                        if (res == 2) res = 3; // NaN input must raise here as well
                    } catch (const std::domain_error&) {
                        if (res != 2) res = 3;
                    } catch (...) {
                        res = 3;
                    }
                    outcome[t] = res;
                    cudaFree(din);
                    cudaFree(dout);
                    if (!use_per_thread_stream) cudaStreamDestroy(st);
                });
            for (auto& th : pool) th.join();
            for (int t = 0; t < 4; ++t) {
                if (outcome[t] != (t == 2 ? 2 : 1))
                    std::printf("thread isolation: per-thread-stream=%d thread %d outcome %d\n", use_per_thread_stream,
                                t, outcome[t]);
                CHECK(outcome[t] == (t == 2 ? 2 : 1));
            }
        }
    }
    // n beyond the GPU DCT kernels' shared-memory row: a clear invalid_argument at creation
    CHECK(throws<std::invalid_argument>([] { DctPlusPlan(16384, RankOneUpdate::self_loop(1, 1.0), 1e-12); }));
    if (failures == 0) std::printf("ALL OK\n");
    return failures == 0 ? 0 : 1;
}
