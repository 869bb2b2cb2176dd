"""CPU tests of the product's host side: the per-graph setup (host-only plans,
device = -1) is bit-identical to the reference's, the API
mirrors the reference's argument checks and exception classes, and the seeded
signal sources reproduce the reference's Rng."""
import numpy as np
import pytest

import paper_2409_08970_b200 as P
from oracle import checkers as O
from tests.golden_io import kat_cases, load_golden, setup_of

BITWISE = ("lambda", "mu", "z", "a", "sigma", "slot_pass", "slot_idx")


def product_update(u: O.Update):
    if u.kind == 0:
        return P.RankOneUpdate.self_loop(u.i, u.rho)
    if u.kind == 1:
        return P.RankOneUpdate.edge_delta(u.i, u.j, u.rho)
    return P.RankOneUpdate.general(u.v, u.rho)


def assert_setup_bitwise(plan, ref: dict, what: str):
    st = plan.setup()
    for k in BITWISE:
        assert np.array_equal(np.asarray(st[k]), np.asarray(ref[k]).astype(np.asarray(st[k]).dtype)), (what, k)
    assert plan.slow_path() == bool(ref["slow_path"]), what


@pytest.mark.parametrize("cid", [1, 2, 3, 4])
def test_setup_bitwise_equal_to_reference(cid):
    cfg = O.config(cid)
    g = load_golden(f"c{cid}")
    if cfg.progressive:
        for r, u in enumerate(cfg.updates, start=1):
            plan = P.DctPlusPlan(cfg.n, product_update(u), 1e-12, device=-1)
            assert_setup_bitwise(plan, setup_of(g, f"m{r}_"), f"C{cid} member {r}")
    else:
        plan = P.DctPlusPlan(cfg.n, product_update(cfg.updates[0]), 1e-12, device=-1)
        assert_setup_bitwise(plan, setup_of(g), f"C{cid}")


@pytest.mark.slow
def test_setup_bitwise_equal_to_reference_c5():
    cfg = O.config(5)
    g = load_golden("c5")
    assert np.array_equal(np.asarray(cfg.updates[0].v), g["v"])
    plan = P.DctPlusPlan(cfg.n, product_update(cfg.updates[0]), 1e-12, device=-1)
    assert_setup_bitwise(plan, setup_of(g), "C5")


def test_setup_bitwise_on_reference_kat_cases():
    for case in kat_cases():
        kind, rho, i, j = case["update"]
        u = O.Update(int(kind), float(rho), int(i), int(j))
        plan = P.DctPlusPlan(int(case["n"]), product_update(u), 1e-12, device=-1)
        assert_setup_bitwise(plan, case, case["name"])


def test_basis_is_orthonormal_and_signed():
    plan = P.DctPlusPlan(32, P.RankOneUpdate.edge_delta(3, 5, 1.5), 1e-12, device=-1)
    x = plan.basis()
    assert np.abs(x.T @ x - np.eye(32)).max() < 1e-10  # acceptance.cpp criterion 3
    # largest-magnitude entry of every column is positive (spectral.hpp:30-37)
    idx = np.abs(x).argmax(axis=0)
    assert np.all(x[idx, np.arange(32)] > 0)


def test_general_update_matches_edge_update():
    n = 16
    v = np.zeros(n)
    v[2], v[4] = 1.0, -1.0
    a = P.DctPlusPlan(n, P.RankOneUpdate.general(v, 1.5), 1e-12, device=-1).setup()
    b = P.DctPlusPlan(n, P.RankOneUpdate.edge_delta(3, 5, 1.5), 1e-12, device=-1).setup()
    for k in BITWISE:
        assert np.array_equal(a[k], b[k]), k


def test_argument_errors_mirror_reference():
    # fast_transform.hpp:52-53, :266-269; graph.hpp:95-108
    with pytest.raises(P.InvalidArgument):
        P.DctPlusPlan(1, P.RankOneUpdate.self_loop(1, 1.0), 1e-12, device=-1)
    with pytest.raises(P.InvalidArgument):
        P.DctPlusPlan(8, P.RankOneUpdate.self_loop(1, 1.0), 2.0, device=-1)
    with pytest.raises(P.InvalidArgument):
        P.DctPlusPlan(8, P.RankOneUpdate.self_loop(1, 1.0), 0.0, device=-1)
    with pytest.raises(P.InvalidArgument):
        P.DctPlusPlan(8, P.RankOneUpdate.self_loop(9, 1.0), 1e-12, device=-1)
    with pytest.raises(P.InvalidArgument):
        P.RankOneUpdate.self_loop(0, 1.0)
    with pytest.raises(P.InvalidArgument):
        P.RankOneUpdate.edge_delta(3, 3, 1.0)
    with pytest.raises(P.InvalidArgument):
        P.RankOneUpdate.edge_delta(1, 2, 0.0)
    with pytest.raises(P.InvalidArgument):
        P.DctPlusPlan(8, P.RankOneUpdate.general(np.ones(7), 1.0), 1e-12, device=-1)
    with pytest.raises(ValueError):  # InvalidArgument is a ValueError
        P.DctPlusPlan(8, P.RankOneUpdate.edge_delta(1, 9, 1.0), 1e-12, device=-1)
    plan = P.DctPlusPlan(8, P.RankOneUpdate.self_loop(1, 1.0), 1e-12, device=-1)
    with pytest.raises(P.InvalidArgument):  # host-only plan cannot apply
        plan.forward(np.zeros(8))
    with pytest.raises(P.InvalidArgument):
        P.PrunedEnsemblePlan(8, [P.RankOneUpdate.self_loop(1, 1.0)], 0, 1.0, device=-1)
    with pytest.raises(P.InvalidArgument):
        P.PrunedEnsemblePlan(8, [P.RankOneUpdate.self_loop(1, 1.0)], 9, 1.0, device=-1)


def test_disconnecting_edge_takes_slow_path_like_reference():
    # test_fast_transform.cpp:259-278: removing an edge of the path trips the guard
    case = next(c for c in kat_cases() if c["name"] == "disconnect_n16")
    plan = P.DctPlusPlan(16, P.RankOneUpdate.edge_delta(8, 9, -1.0), 1e-12, device=-1)
    assert plan.slow_path() == bool(case["slow_path"]) == True  # noqa: E712


def test_ensemble_members_host_only():
    ws = [0.05 + k * (1.95 / 15.0) for k in range(16)]
    ens = P.PrunedEnsemblePlan(128, [P.RankOneUpdate.self_loop(1, w) for w in ws], 128, 1e300, device=-1)
    assert ens.ensemble_size() == 17 and ens.size() == 128 and ens.keep_count() == 128
    g = load_golden("c4")
    for r in (1, 8, 16):
        assert_setup_bitwise(ens.member(r), setup_of(g, f"m{r}_"), f"member {r}")
    with pytest.raises(P.LogicError):
        ens.member(0)
    with pytest.raises(P.LogicError):
        ens.member(17)


@pytest.mark.parametrize("dist,r", [(0, 0.0), (1, 0.0), (2, 0.95), (3, 0.0), (4, 0.9)])
def test_signal_sources_match_oracle(restatement, dist, r):
    a = P.fill_signals(77, dist, 128, 300, r)
    b = restatement.fill_signals(77, dist, 128, 300, r)
    assert np.array_equal(a, b)


def test_signal_sources_match_reference_goldens():
    for cid in (1, 2, 3, 4):
        g = load_golden(f"c{cid}")
        s = P.fill_signals(int(g["seed"]), int(g["dist"]), int(g["n"]), g["signals"].shape[0], float(g["r"]))
        assert np.array_equal(s, g["signals"])
    assert P.mix_seed(2409, 1024, 3) == O.mix_seed(2409, 1024, 3)


def test_pruned_ensemble_constructs_host_only():
    """c_p < n (the pruned mode, fast_transform.hpp:343-375) builds on the host
    like c_p = n; applying a host-only ensemble is an InvalidArgument."""
    ups = [P.RankOneUpdate.self_loop(1, 1.5), P.RankOneUpdate.edge_delta(2, 3, 1.5)]
    ens = P.PrunedEnsemblePlan(32, ups, 16, 0.5, device=-1)
    assert ens.keep_count() == 16 and ens.threshold() == 0.5 and ens.ensemble_size() == 3
    with pytest.raises(P.InvalidArgument):
        ens.forward_all(np.zeros(32))


@pytest.mark.parametrize("n,r,quantile,seed", [(32, 0.99, 0.7, 42), (128, 0.95, 0.5, 7), (16, 0.9, 0.9, 1)])
def test_calibrate_prune_threshold_matches_reference(reference, n, r, quantile, seed):
    """bench.hpp:99-108 on the reference's Rng: bit-identical threshold."""
    ours = P.calibrate_prune_threshold(n, r, quantile, 512, seed)
    ref = reference.lib.ref_calibrate_prune_threshold(n, r, quantile, 512, seed)
    assert ours == ref


# --- rank-k chains (cauchy.hpp:159-231) -----------------------------------------

CHAIN_CASES = [
    (8, [O.Update(0, 1.5, 1)]),
    (8, [O.Update(0, 1.5, 1), O.Update(0, 0.8, 8)]),
    (8, [O.Update(0, 0.9, 2), O.Update(0, -0.9, 2)]),
    (64, [O.Update(1, -0.5, 1, 64), O.Update(0, 2.0, 3), O.Update(1, 0.7, 5, 9)]),
    (100, [O.Update(1, 1.0, 1, 100), O.Update(1, 1.0, 1, 100)]),  # stage 2 deflates by rotations
    (48, [O.Update(2, 0.6, v=tuple(np.cos(np.arange(48) * 0.3))), O.Update(0, -1.2, 7)]),
]


def path_laplacian(n, ups):
    lap = np.zeros((n, n))
    for i in range(n - 1):
        lap[i, i] += 1.0
        lap[i + 1, i + 1] += 1.0
        lap[i, i + 1] -= 1.0
        lap[i + 1, i] -= 1.0
    for u in ups:
        v = O.direction(u, n)
        lap += u.rho * np.outer(v, v)
    return lap


@pytest.mark.parametrize("case", range(len(CHAIN_CASES)))
def test_chain_compose_bitwise_equal_to_reference(reference, case):
    """compose_rank_k's final basis and eigenvalues are the reference's, bit
    for bit (host-only chain), including a stage that deflates by Givens
    rotations and a general-direction stage."""
    n, ups = CHAIN_CASES[case]
    ch = P.compose_rank_k(n, [product_update(u) for u in ups], device=-1)
    mu, x, k = reference.chain(n, ups).spectrum()
    assert k == len(ups) == len(ch.stages)
    assert np.array_equal(ch.mu, mu)
    assert np.array_equal(ch.x, x)


def test_chain_compose_on_a_caller_base_matches_reference(reference):
    """A non-path base spectrum (dense eigendecomposition of a perturbed path)
    composes bit-identically too."""
    n = 24
    lam, u = np.linalg.eigh(path_laplacian(n, [O.Update(0, 0.7, 5)]))
    ups = [O.Update(1, 0.4, 2, 20), O.Update(0, -0.3, 11)]
    ch = P.compose_rank_k(P.SpectralBasis(lam, u), [product_update(v) for v in ups], device=-1)
    mu, x, _ = reference.chain(n, ups, base=(lam, u)).spectrum()
    assert np.array_equal(ch.mu, mu) and np.array_equal(ch.x, x)


def test_chain_k1_reduces_to_the_plan_and_k2_to_the_dense_oracle():
    """test_cauchy.cpp:203-247: k = 1 gives the plan's spectrum; k = 2 the
    dense eigendecomposition; a cancelling pair returns the base spectrum."""
    n = 8
    plan = P.DctPlusPlan(n, P.RankOneUpdate.self_loop(1, 1.5), 1e-12, device=-1)
    ch = P.compose_rank_k(n, [P.RankOneUpdate.self_loop(1, 1.5)], device=-1)
    assert np.max(np.abs(ch.mu - plan.mu())) < 1e-14
    assert np.max(np.abs(np.abs(ch.x) - np.abs(plan.basis()))) < 1e-12
    ups = [O.Update(0, 1.5, 1), O.Update(0, 0.8, n)]
    ch = P.compose_rank_k(n, [product_update(u) for u in ups], device=-1)
    lam = np.linalg.eigvalsh(path_laplacian(n, ups))
    assert np.max(np.abs(ch.mu - lam)) < 1e-8
    ch = P.compose_rank_k(n, [P.RankOneUpdate.self_loop(2, 0.9), P.RankOneUpdate.self_loop(2, -0.9)], device=-1)
    assert np.max(np.abs(ch.mu - P.path_spectrum(n).lambda_)) < 1e-8


def test_chain_errors_mirror_reference():
    with pytest.raises(P.InvalidArgument, match="need k >= 1"):
        P.compose_rank_k(4, [], device=-1)
    with pytest.raises(P.RuntimeFailure, match="stage 2"):
        P.compose_rank_k(8, [P.RankOneUpdate.self_loop(1, 1.5), P.RankOneUpdate.self_loop(99, 1.0)], device=-1)
    ch = P.compose_rank_k(8, [P.RankOneUpdate.self_loop(1, 1.5)], device=-1)
    with pytest.raises(P.InvalidArgument, match="host-only"):
        ch.forward(np.zeros(8))


def test_host_only_plan_route_query():
    """dctp_plan_route on a host-only plan (no device constants): no NFST
    route and no creation probe (the probe needs the GPU)."""
    import paper_2409_08970_b200 as P

    plan = P.DctPlusPlan(1024, P.RankOneUpdate.self_loop(1, 0.5), 1e-12, device=-1)
    assert plan.route() == {"nfst": False, "probe_gap": 0.0}
    assert not plan.slow_path()
