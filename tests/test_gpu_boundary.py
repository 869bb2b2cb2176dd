"""Boundary behaviour on the GPU: caller-supplied outputs are validated,
per-thread non-finite flags, the tcgen05 GEMM's row slicing beyond the grid
limit, the DCT size limit, and the int8 (Ozaki) product's slice-count knob."""
import os
import subprocess
import sys
import threading
from pathlib import Path

import numpy as np
import pytest

from oracle import checkers as O

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def P():
    import paper_2409_08970_b200 as P

    return P


@pytest.fixture(scope="module")
def torch():
    import torch

    torch.cuda.init()
    return torch


def test_out_argument_is_validated(P, torch):
    plan = P.DctPlusPlan(64, P.RankOneUpdate.self_loop(1, 0.5), 1e-12)
    x = torch.randn((10, 64), dtype=torch.float64, device="cuda")
    good = torch.empty_like(x)
    assert plan.forward(x, out=good) is not None
    bad = [torch.empty((10, 64), dtype=torch.float32, device="cuda"),   # dtype
           torch.empty((9, 64), dtype=torch.float64, device="cuda"),    # short
           torch.empty((64, 10), dtype=torch.float64, device="cuda").t(),  # strided view
           torch.empty((10, 64), dtype=torch.float64),                  # host
           x]                                                            # aliasing the input
    for out in bad:
        with pytest.raises(P.InvalidArgument):
            plan.forward(x, out=out)
    # one signal: out without the batch axis is accepted
    y1 = torch.empty(64, dtype=torch.float64, device="cuda")
    plan.forward(x[0], out=y1)
    assert torch.allclose(y1, plan.forward(x[0]))
    ens = P.PrunedEnsemblePlan(64, [P.RankOneUpdate.self_loop(1, w) for w in (0.5, 1.0)], 64, 1.7e308)
    with pytest.raises(P.InvalidArgument):
        ens.forward_all_batch(x, out=torch.empty((10, 2, 64), dtype=torch.float64, device="cuda"))


def test_nan_surfaces_only_in_its_own_thread(P, torch):
    """Four host threads share one plan, each on its own stream; only the
    thread whose batch holds a NaN gets DomainError (fast_transform.hpp:33-34,
    271-276: the failing call throws)."""
    plan = P.DctPlusPlan(256, P.RankOneUpdate.edge_delta(128, 129, -0.7), 1e-12)
    base = torch.as_tensor(P.fill_signals(3, P.DIST_AR, 256, 1024, 0.95), device="cuda")
    results = [None] * 4
    barrier = threading.Barrier(4)

    def work(t):
        s = torch.cuda.Stream()
        x = base.clone()
        if t == 1:
            x[500, 7] = float("nan")
        torch.cuda.synchronize()
        barrier.wait()
        out = "ok"
        with torch.cuda.stream(s):
            for _ in range(10):
                try:
                    plan.forward(x)
                except P.DomainError:
                    out = "domain"
                    break
        results[t] = out

    th = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert results == ["ok", "domain", "ok", "ok"], results


def test_tc_sgemm_row_slices_match_single_grid(P, torch, tmp_path):
    """The tcgen05 3xTF32 GEMM launches row slices once the row tiles exceed
    the grid limit; a lowered slice size (3 tiles) must give bit-identical
    C4 outputs."""
    script = tmp_path / "c4.py"
    script.write_text(
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {str(ROOT)!r})\n"
        "import paper_2409_08970_b200 as P\n"
        "ws = [0.05 + k * (1.95 / 15.0) for k in range(16)]\n"
        "ens = P.PrunedEnsemblePlan(128, [P.RankOneUpdate.self_loop(1, w) for w in ws], 128, 1.7e308)\n"
        "x = torch.as_tensor(P.fill_signals(P.mix_seed(2409, 128, 4), P.DIST_AR2D, 128, 5000, 0.9), device='cuda')\n"
        "np.save(sys.argv[1], ens.forward_all_batch(x.float()).cpu().numpy())\n")
    outs = []
    for tiles in ("65535", "3"):
        f = tmp_path / f"y{tiles}.npy"
        env = dict(os.environ, DCTP_TC32_SLICE_TILES=tiles)
        subprocess.run([sys.executable, str(script), str(f)], env=env, check=True, timeout=300)
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


def test_dct_size_limit_is_a_clear_error(P, torch):
    with pytest.raises(P.InvalidArgument, match="exceeds the GPU DCT kernels"):
        P.DctPlusPlan(16384, P.RankOneUpdate.self_loop(1, 1.0), 1e-12)
    with pytest.raises(P.InvalidArgument):
        P.dct2(torch.zeros((1, 16384), dtype=torch.float64, device="cuda"))


def test_ozaki_slice_counts_agree(P, torch, reference, tmp_path):
    """DCTP_OZAKI_SLICES=6 (21 int8 products) and the default 5 (15) both
    meet the fp64 tolerance on a general-direction dense plan; 6 is ~100x
    tighter."""
    script = tmp_path / "oz.py"
    script.write_text(
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {str(ROOT)!r})\n"
        "import paper_2409_08970_b200 as P\n"
        "n = 2048\n"
        "v = P.fill_signals(P.mix_seed(2409, n, 50), 0, n, 1)[0] / np.sqrt(n)\n"
        "plan = P.DctPlusPlan(n, P.RankOneUpdate.general(v, 0.1), 1e-12)\n"
        "assert P.ozaki_slices(n) == int(sys.argv[2])\n"
        "x = torch.as_tensor(P.fill_signals(5, 0, n, 300), device='cuda')\n"
        "np.save(sys.argv[1], plan.forward(x).cpu().numpy())\n")
    n = 2048
    v = P.fill_signals(P.mix_seed(2409, n, 50), 0, n, 1)[0] / np.sqrt(n)
    want = reference.plan(n, O.Update(2, 0.1, 0, 0, tuple(v))).forward(P.fill_signals(5, 0, n, 300))
    errs = {}
    for sl in ("5", "6"):
        f = tmp_path / f"y{sl}.npy"
        env = dict(os.environ, DCTP_OZAKI_SLICES=sl)
        subprocess.run([sys.executable, str(script), str(f), sl], env=env, check=True, timeout=300)
        errs[sl] = O.parity(np.load(f), want)
    assert errs["5"] <= 1e-10 and errs["6"] <= 1e-12, errs


def test_ozaki_persistent_split_and_one_tile_kernels_agree(P, torch, reference, tmp_path):
    """The int8 products' three schedules give bit-identical coefficients:
    the persistent CTA-pair kernel (K <= 2048) with its split-K tail (1000
    rows of n = 2048: 4 pairs x 22 column tiles on 74 pair slots leave a
    14-tile tail split 4 ways), the same kernel unsplit (DCTP_OZAKI_SPLIT=0)
    and the one-tile pair kernel (DCTP_OZAKI_PERSIST=0) — exact int32 level
    sums, the same Horner and scaling order — for 5 slices (96-column tiles)
    and 6 (80-column tiles); and the default meets the fp64 tolerance
    against the reference."""
    script = tmp_path / "ozp.py"
    script.write_text(
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {str(ROOT)!r})\n"
        "import paper_2409_08970_b200 as P\n"
        "n = 2048\n"
        "v = P.fill_signals(P.mix_seed(2409, n, 50), 0, n, 1)[0] / np.sqrt(n)\n"
        "plan = P.DctPlusPlan(n, P.RankOneUpdate.general(v, 0.1), 1e-12)\n"
        "x = torch.as_tensor(P.fill_signals(7, 0, n, 1000), device='cuda')\n"
        "np.save(sys.argv[1], plan.forward(x).cpu().numpy())\n")
    n = 2048
    v = P.fill_signals(P.mix_seed(2409, n, 50), 0, n, 1)[0] / np.sqrt(n)
    want = reference.plan(n, O.Update(2, 0.1, 0, 0, tuple(v))).forward(P.fill_signals(7, 0, n, 1000))
    for sl in ("5", "6"):
        outs = {}
        for mode, extra in (("split", {}), ("unsplit", {"DCTP_OZAKI_SPLIT": "0"}),
                            ("one_tile", {"DCTP_OZAKI_PERSIST": "0"})):
            f = tmp_path / f"y{sl}_{mode}.npy"
            env = dict(os.environ, DCTP_OZAKI_SLICES=sl, **extra)
            subprocess.run([sys.executable, str(script), str(f)], env=env, check=True, timeout=300)
            outs[mode] = np.load(f)
        assert np.array_equal(outs["split"], outs["unsplit"]), sl
        assert np.array_equal(outs["split"], outs["one_tile"]), sl
        assert O.parity(outs["split"], want) <= 1e-10


def test_grouped_int8_fold_route_matches_reference(P, torch, reference, tmp_path):
    """The opt-in grouped int8 route of small folded plans (DCTP_FOLD_I8=1:
    the [y | u] slicing pass and the persistent CTA-pair product with even /
    odd column-tile groups) meets the fp64 tolerance against the reference on
    a ragged C2-shape batch and agrees with the default fused kernel."""
    script = tmp_path / "fi8.py"
    script.write_text(
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {str(ROOT)!r})\n"
        "import paper_2409_08970_b200 as P\n"
        "plan = P.DctPlusPlan(256, P.RankOneUpdate.edge_delta(128, 129, -0.7), 1e-12)\n"
        "x = torch.as_tensor(P.fill_signals(13, P.DIST_AR, 256, 1001, 0.95), device='cuda')\n"
        "np.save(sys.argv[1], plan.forward(x).cpu().numpy())\n")
    outs = {}
    for mode in ("0", "1"):
        f = tmp_path / f"y{mode}.npy"
        subprocess.run([sys.executable, str(script), str(f)], env=dict(os.environ, DCTP_FOLD_I8=mode), check=True,
                       timeout=300)
        outs[mode] = np.load(f)
    want = reference.plan(256, O.Update(1, -0.7, 128, 129)).forward(P.fill_signals(13, P.DIST_AR, 256, 1001, 0.95))
    assert O.parity(outs["1"], want) <= 1e-10
    assert O.parity(outs["1"], outs["0"]) <= 1e-10


def test_cuda_graph_capture_and_replay(P, torch):
    """Launches captured into a CUDA graph replay to the same coefficients;
    a non-finite sample fed through the graph raises DomainError at the next
    sync_check (the object's graph flag)."""
    plan = P.DctPlusPlan(256, P.RankOneUpdate.edge_delta(128, 129, -0.7), 1e-12)
    x = torch.as_tensor(P.fill_signals(9, P.DIST_AR, 256, 2048, 0.95), device="cuda")
    want = plan.forward(x)
    y = torch.empty_like(x)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        plan.forward(x, sync=False, out=y)  # warm-up outside the capture
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            plan.forward(x, sync=False, out=y)
    y.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, want)
    x[3, 4] = float("nan")
    g.replay()
    with pytest.raises(P.DomainError):
        plan.sync_check()
    plan.sync_check()  # cleared
