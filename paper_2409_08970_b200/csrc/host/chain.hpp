// Rank-k chains: L + sum_r rho_r v_r v_r^T as k successive rank-one stages
// (compose_rank_k, proj/include/dctplus/cauchy.hpp:159-216).
//
// The host composes the chain once, op-for-op like the reference (each
// stage's z against the materialised previous basis, the deflation's Givens
// rotations applied to it, the unsigned basis assembled column by column,
// signs fixed per column), so the final basis X and eigenvalues mu are
// bit-identical to the reference's.  The batched apply (chain_forward,
// cauchy.hpp:218-231, which runs U^T s and then k Cauchy stages) is then a
// single product with X on the device: k Cauchy stages of n^2 terms each
// cost k times the one dense n x n product, which on the tensor cores also
// drops every per-entry division.  Same -ffp-contract=off rule as setup.hpp.
#pragma once

#include <cmath>
#include <cstddef>
#include <numbers>
#include <stdexcept>
#include <string>
#include <vector>

#include "host/setup.hpp"

namespace dctp::host {

struct ChainStage {
    std::vector<double> base_vals; // spectrum entering the stage
    Perturbed spec;
    std::vector<double> sigma;
};

struct Chain {
    std::size_t n = 0;
    std::vector<double> base_lambda, base_u; // base_u row-major n x n, column k = eigenvector k
    std::vector<ChainStage> stages;
    std::vector<double> x, mu; // final signed basis (row-major), final eigenvalues (ascending)
};

/// path_spectrum (spectral.hpp:48-68): lambda_k = 2 - 2 cos(k pi / n) and
/// the orthonormal DCT-II basis, evaluated with the reference's expression
/// order.
inline void path_spectrum(std::size_t n, std::vector<double>& lambda, std::vector<double>& u) {
    if (n < 2) throw std::invalid_argument("path_spectrum: need n >= 2");
    const double pi = std::numbers::pi;
    const double nd = static_cast<double>(n);
    const double scale = std::sqrt(2.0 / nd);
    lambda.assign(n, 0.0);
    u.assign(n * n, 0.0);
    for (std::size_t k = 0; k < n; ++k) {
        lambda[k] = 2.0 - 2.0 * std::cos(static_cast<double>(k) * pi / nd);
        const double ck = (k == 0) ? 1.0 / std::numbers::sqrt2 : 1.0;
        for (std::size_t j = 0; j < n; ++j)
            u[j * n + k] =
                ck * scale * std::cos(pi * static_cast<double>(k) * (2.0 * static_cast<double>(j) + 1.0) / (2.0 * nd));
    }
    lambda[0] = 0.0;
}

namespace chain_detail {

/// z = U^T v, accumulated row by row (matrix.hpp:71-79).
inline std::vector<double> matvec_t(const std::vector<double>& u, std::size_t n, const std::vector<double>& v) {
    std::vector<double> y(n, 0.0);
    for (std::size_t i = 0; i < n; ++i) {
        const double xi = v[i];
        for (std::size_t j = 0; j < n; ++j) y[j] += u[i * n + j] * xi;
    }
    return y;
}

/// The deflation's rotations applied to the basis columns (cauchy.hpp:57-68).
inline std::vector<double> rotated_basis(const std::vector<double>& u, std::size_t n,
                                         const std::vector<Rotation>& rots) {
    std::vector<double> r = u;
    for (const Rotation& g : rots)
        for (std::size_t i = 0; i < n; ++i) {
            const double a = r[i * n + g.into], b = r[i * n + g.from];
            r[i * n + g.into] = g.c * a + g.s * b;
            r[i * n + g.from] = -g.s * a + g.c * b;
        }
    return r;
}

/// Signed basis of one stage: column s = U_eff y_s with y_s the pass-through
/// unit vector or a_s z_j / (lambda_j - nu) (cauchy.hpp:84-103), each a
/// left-to-right row dot product (matrix.hpp:59-69), then the column sign
/// convention (spectral.hpp:30-37).  Columns are independent: host threads.
inline std::vector<double> signed_basis(const std::vector<double>& u_eff, const std::vector<double>& lam,
                                        const Perturbed& ps, std::vector<double>& sigma) {
    const std::size_t n = lam.size();
    std::vector<double> x(n * n);
    sigma.assign(n, 1.0);
    parallel_for(n, [&](std::size_t s) {
        std::vector<double> y(n, 0.0), col(n);
        if (ps.slots[s].passthrough) {
            y[ps.slots[s].idx] = 1.0;
        } else {
            const double nu = ps.sub_mu[ps.slots[s].idx];
            for (std::size_t j = 0; j < n; ++j)
                if (ps.z[j] != 0.0) y[j] = ps.a[s] * ps.z[j] / (lam[j] - nu);
        }
        for (std::size_t i = 0; i < n; ++i) {
            double acc = 0.0;
            for (std::size_t j = 0; j < n; ++j) acc += u_eff[i * n + j] * y[j];
            col[i] = acc;
        }
        sigma[s] = sign_of_column(col.data(), n);
        for (std::size_t i = 0; i < n; ++i) x[i * n + s] = sigma[s] < 0.0 ? -col[i] : col[i];
    }, 2);
    return x;
}

} // namespace chain_detail

/// compose_rank_k (cauchy.hpp:175-216).  An empty base means path_spectrum(n).
inline Chain compose_rank_k(std::size_t n, const std::vector<Update>& updates, std::vector<double> base_lambda,
                            std::vector<double> base_u, double tau) {
    if (updates.empty()) throw std::invalid_argument("compose_rank_k: need k >= 1 updates");
    Chain ch;
    ch.n = n;
    if (base_lambda.empty() && base_u.empty()) {
        path_spectrum(n, ch.base_lambda, ch.base_u);
    } else {
        if (n < 1 || base_lambda.size() != n || base_u.size() != n * n)
            throw std::invalid_argument("compose_rank_k: base spectrum dimension mismatch");
        ch.base_lambda = std::move(base_lambda);
        ch.base_u = std::move(base_u);
    }
    std::vector<double> cur_u = ch.base_u, cur_vals = ch.base_lambda;
    for (std::size_t r = 0; r < updates.size(); ++r) {
        try {
            const std::vector<double> v = updates[r].direction(n);
            const std::vector<double> z = chain_detail::matvec_t(cur_u, n, v);
            ChainStage st;
            st.base_vals = cur_vals;
            st.spec = perturb_spectrum(cur_vals, z, updates[r].rho, tau);
            const std::vector<double> u_eff = chain_detail::rotated_basis(cur_u, n, st.spec.rotations);
            std::vector<double> x = chain_detail::signed_basis(u_eff, st.base_vals, st.spec, st.sigma);
            cur_vals = st.spec.mu;
            cur_u = std::move(x);
            ch.stages.push_back(std::move(st));
        } catch (const std::exception& e) {
            throw std::runtime_error("compose_rank_k: stage " + std::to_string(r + 1) + ": " + e.what());
        }
    }
    ch.x = std::move(cur_u);
    ch.mu = std::move(cur_vals);
    return ch;
}

} // namespace dctp::host
