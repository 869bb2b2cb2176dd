"""Guard-band memory-safety checks of every kernel family (compute-sanitizer
is closed on this GPU pool, profiles/r02/sanitizer_closed.txt).

Each apply writes into a view in the middle of a larger buffer whose guard
rows (before and after) hold a sentinel; after the call the guards must be
intact, the view fully written (no sentinel left), the input unchanged, and
the result equal to a plain call's.  Batches are ragged (1, a few, one past
a tile, one short of a tile pair) so the kernels' partial tiles and padded
rows are exercised at both ends of the output.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SENTINEL = 7.77e7
GUARD = 3  # guard rows on each side


@pytest.fixture(scope="module")
def P():
    import paper_2409_08970_b200 as P

    return P


@pytest.fixture(scope="module")
def torch():
    import torch

    torch.cuda.init()
    return torch


def _guarded(torch, shape, dtype):
    """A buffer of GUARD + rows + GUARD rows filled with the sentinel, and
    the contiguous view of its middle rows."""
    full = torch.full((shape[0] + 2 * GUARD, *shape[1:]), SENTINEL, dtype=dtype, device="cuda")
    return full, full[GUARD:GUARD + shape[0]]


def _check(torch, full, view, want, x, x0):
    torch.cuda.synchronize()
    head, tail = full[:GUARD], full[GUARD + view.shape[0]:]
    assert bool((head == SENTINEL).all()), "write before the output rows"
    assert bool((tail == SENTINEL).all()), "write past the output rows"
    assert not bool((view == SENTINEL).any()), "output element left unwritten"
    assert torch.equal(x, x0), "input modified"
    assert torch.equal(view, want), "guarded output differs from a plain call"


def _signals(P, torch, n, rows, dtype, seed=11):
    return torch.as_tensor(P.fill_signals(seed, 0, n, rows), device="cuda").to(dtype)


# (n, update, dtypes, ops): one plan per kernel family / route
CASES = {
    "small_dense_n64": (64, ("self_loop", 1, 0.5), ("f64", "f32"), ("forward", "inverse")),
    "fused_pingpong_n256": (256, ("edge_delta", 128, 129, -0.7), ("f64", "f32"), ("forward", "inverse")),
    "fold_n1024": (1024, ("edge_delta", 1, 1024, 1.0), ("f64", "f32"), ("forward", "inverse")),
    "nfst_n1024": (1024, ("self_loop", 1, 0.5), ("f64",), ("forward", "inverse")),
    "selfloop_n512": (512, ("self_loop", 1, 2.0), ("f64", "f32"), ("forward", "inverse")),  # NFST / structured routes
}


def _update(P, spec):
    kind, *args = spec
    return getattr(P.RankOneUpdate, kind)(*args)


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("rows", [1, 5, 129, 255])
def test_guard_rows_intact(P, torch, case, rows):
    n, spec, dtypes, ops = CASES[case]
    plan = P.DctPlusPlan(n, _update(P, spec), 1e-12)
    for dt in dtypes:
        dtype = torch.float64 if dt == "f64" else torch.float32
        x = _signals(P, torch, n, rows, dtype)
        x0 = x.clone()
        for op in ops:
            fn = plan.forward if op == "forward" else plan.inverse
            want = fn(x)
            full, view = _guarded(torch, (rows, n), dtype)
            fn(x, out=view)
            _check(torch, full, view, want, x, x0)


@pytest.mark.parametrize("rows", [1, 7, 300])
def test_guard_rows_dense_int8(P, torch, rows):
    """The dense route of a general direction at n = 1024: the int8 slicing
    pass and the CTA-pair tensor-core product (forward X^T s, inverse X p)."""
    n = 1024
    v = P.fill_signals(P.mix_seed(2409, n, 50), 0, n, 1)[0] / np.sqrt(n)
    plan = P.DctPlusPlan(n, P.RankOneUpdate.general(v, 0.1), 1e-12)
    x = _signals(P, torch, n, rows, torch.float64)
    x0 = x.clone()
    for fn in (plan.forward, plan.inverse):
        want = fn(x)
        full, view = _guarded(torch, (rows, n), torch.float64)
        fn(x, out=view)
        _check(torch, full, view, want, x, x0)


@pytest.mark.parametrize("rows", [1, 129, 300])
@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_guard_rows_progressive(P, torch, rows, dt):
    """forward_all of the C4 ensemble (n = 128, K = 16): the persistent
    bf16x3 GEMM (fp32) and the DCT + Cauchy stages (fp64); (rows, 17, n)."""
    n = 128
    ws = [0.05 + k * (1.95 / 15.0) for k in range(16)]
    ens = P.PrunedEnsemblePlan(n, [P.RankOneUpdate.self_loop(1, w) for w in ws], n, 1.7e308)
    dtype = torch.float64 if dt == "f64" else torch.float32
    x = _signals(P, torch, n, rows, dtype)
    x0 = x.clone()
    want = ens.forward_all_batch(x)
    full, view = _guarded(torch, (rows, 17, n), dtype)
    ens.forward_all_batch(x, out=view)
    _check(torch, full, view, want, x, x0)


@pytest.mark.parametrize("rows", [1, 33, 300])
def test_guard_rows_chain(P, torch, rows):
    """A rank-3 chain at n = 1024 (X6's shape): the composed basis product."""
    n = 1024
    ups = [P.RankOneUpdate.self_loop(1, 1.5), P.RankOneUpdate.edge_delta(1, 1024, -0.5),
           P.RankOneUpdate.edge_delta(300, 700, 0.25)]
    chain = P.ChainedFactorization(P.path_spectrum(n), ups)
    x = _signals(P, torch, n, rows, torch.float64)
    x0 = x.clone()
    want = chain.forward(x)
    full, view = _guarded(torch, (rows, n), torch.float64)
    chain.forward(x, out=view)
    _check(torch, full, view, want, x, x0)
