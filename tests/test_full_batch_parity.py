"""Full-batch parity: every BASELINE config at its full batch, every signal,
against the reference itself (oracle/_ref — the unmodified headers compiled
in place, run on all host threads with one shared plan and one workspace per
thread, proj/README.md:82-87).

Reference paths (fast_transform.hpp): DctPlusPlan::forward (:163-195; the
fast route for C1/C2, the dense X^T s for C3/C5 whose near-pole guard trips),
DctPlusPlan::inverse (:218-260), PrunedEnsemblePlan::forward_all with
c_p = n (:396-439, all K + 1 sets: the C4 oracle).

Tolerance (north star), norm-wise per signal,
e = max_i |y_i - r_i| / max_i |r_i|, max over the whole batch:
    fp64 <= 1e-10,  fp32 <= 1e-4 (against the fp64 reference).
Inputs: the reference's Rng seeded mix_seed(2409, n, config) — the product
draws bit-identical signals (tests/test_host_setup.py)."""
import numpy as np
import pytest

from oracle import checkers as O

pytestmark = pytest.mark.gpu

TOL64, TOL32 = 1e-10, 1e-4
THREADS = 0  # all host threads


@pytest.fixture(scope="module")
def P():
    import paper_2409_08970_b200 as P

    return P


@pytest.fixture(scope="module")
def torch():
    import torch

    torch.cuda.init()
    return torch


def _upd(P, u):
    if u.kind == 0:
        return P.RankOneUpdate.self_loop(u.i, u.rho)
    if u.kind == 1:
        return P.RankOneUpdate.edge_delta(u.i, u.j, u.rho)
    return P.RankOneUpdate.general(u.v, u.rho)


_cache = {}


def _case(P, reference, cid):
    """(config, GPU plan, reference plan, full-batch signals), built once."""
    if cid not in _cache:
        cfg = O.config(cid)
        s = reference.fill(cfg.seed, cfg.dist, cfg.n, cfg.batch, cfg.r)
        if cfg.progressive:
            plan = P.PrunedEnsemblePlan(cfg.n, [_upd(P, u) for u in cfg.updates], cfg.n, 1.7e308)
            rp = reference.ensemble(cfg.n, list(cfg.updates), cfg.n, float(np.finfo(np.float64).max))
        else:
            plan = P.DctPlusPlan(cfg.n, _upd(P, cfg.updates[0]), 1e-12)
            rp = reference.plan(cfg.n, cfg.updates[0])
        _cache[cid] = (cfg, plan, rp, s, {})
    return _cache[cid]


def _ref_forward(case):
    cfg, plan, rp, s, memo = case
    if "fwd" not in memo:
        memo["fwd"] = rp.forward_all(s, threads=THREADS) if cfg.progressive else rp.forward(s, threads=THREADS)
    return memo["fwd"]


def _dev(torch, a, dtype):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda").to(dtype)


@pytest.mark.parametrize("cid,dtype", [(1, "float64"), (1, "float32"), (2, "float64"), (2, "float32"),
                                       (3, "float64"), (3, "float32"), (5, "float64")])
def test_forward_full_batch_against_reference(P, torch, reference, cid, dtype):
    case = _case(P, reference, cid)
    cfg, plan, _, s, _ = case
    want = _ref_forward(case)
    got = plan.forward(_dev(torch, s, getattr(torch, dtype))).double().cpu().numpy()
    assert got.shape == (cfg.batch, cfg.n)
    assert O.parity(got, want) <= (TOL64 if dtype == "float64" else TOL32)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_inverse_c3_full_batch_against_reference(P, torch, reference, dtype):
    """C3 inverse: p = the reference's own forward coefficients of the whole
    batch, s = inverse(p) against DctPlusPlan::inverse (:218-260)."""
    case = _case(P, reference, 3)
    cfg, plan, rp, s, memo = case
    p = _ref_forward(case)
    if "inv" not in memo:
        memo["inv"] = rp.inverse(p, threads=THREADS)
    got = plan.inverse(_dev(torch, p, getattr(torch, dtype))).double().cpu().numpy()
    assert O.parity(got, memo["inv"]) <= (TOL64 if dtype == "float64" else TOL32)


def test_inverse_c5_full_batch_against_reference(P, torch, reference):
    case = _case(P, reference, 5)
    cfg, plan, rp, s, memo = case
    p = _ref_forward(case)
    want = rp.inverse(p, threads=THREADS)
    got = plan.inverse(_dev(torch, p, torch.float64)).cpu().numpy()
    assert O.parity(got, want) <= TOL64


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_progressive_c4_full_batch_all_sets(P, torch, reference, dtype):
    """All 65536 signals, all 17 sets (set 0 = the shared DCT) against the
    reference's forward_all with c_p = n."""
    case = _case(P, reference, 4)
    cfg, plan, _, s, _ = case
    want = _ref_forward(case)
    got = plan.forward_all_batch(_dev(torch, s, getattr(torch, dtype))).double().cpu().numpy()
    assert got.shape == want.shape == (cfg.batch, 17, cfg.n)
    tol = TOL64 if dtype == "float64" else TOL32
    for r in range(17):
        assert O.parity(got[:, r, :], want[:, r, :]) <= tol, r


def test_full_batch_slot_order_and_signs(P, torch, reference):
    """Sign flips or slot permutations would hide from norm properties; the
    per-slot comparison above sees them — here the setup itself: mu and
    sigma of every config bit-identical to the reference's."""
    for cid in (1, 2, 3, 5):
        case = _case(P, reference, cid)
        cfg, plan, rp, _, _ = case
        mine, theirs = plan.setup(), rp.setup()
        assert np.array_equal(mine["mu"], theirs["mu"]), cid
        assert np.array_equal(mine["sigma"], theirs["sigma"]), cid
        assert np.array_equal(mine["slot_pass"], theirs["slot_pass"]), cid
