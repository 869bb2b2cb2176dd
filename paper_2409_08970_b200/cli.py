"""Benchmark and transform CLI with the reference's CSV contract
(proj/tools/fastdctplus.cpp, proj/include/dctplus/bench.hpp):

    python -m paper_2409_08970_b200.cli accuracy  --sizes 8,16,32 --trials 1000 --out acc.csv
    python -m paper_2409_08970_b200.cli runtime   --sizes 8,...,256 --trials 2000 --out rt.csv
    python -m paper_2409_08970_b200.cli prune     --sizes 32 --cp 16 --threshold 50 --out prune.csv
    python -m paper_2409_08970_b200.cli transform --update selfloop:1:1.5 < signal.txt

CSV rows are `mode,size,update,method,metric,value` with %.6e values and the
same (mode, method, metric) keys, cells, seeds (mix_seed per cell) and signal
sources (gen_ar_signal on the reference Rng) as bench.hpp:176-372, so the
two CSVs line up row for row.  What differs is what a row measures:

* every transform runs on the GPU; `fastdctplus` is the structured route
  (DCT + Cauchy), `nmvp` the dense product with the materialised basis (both
  fp64 tensor-core kernels), `dct` the batched DCT-II kernel;
* runtime `mean_ns` is batched throughput — one launch over all `trials`
  signals of the cell, timed with CUDA events (best of two), divided by the
  trial count — not the reference's one-signal-at-a-time latency;
* prune `direct` is the DCT plus each member's faster route, `pruned_cpN`
  forward_all over the pool, both batched the same way.

The transform subcommand's --graph (dense Jacobi GFT of a general graph
file) is outside this library's scope and is rejected.
"""
from __future__ import annotations

import argparse
import math
import re
import sys
from typing import List, Sequence

import numpy as np

from . import _native as N
from .dctplus import (DIST_AR, DctPlusPlan, PrunedEnsemblePlan, RankOneUpdate, calibrate_prune_threshold, dct2,
                      fill_signals, mix_seed)

CSV_HEADER = "mode,size,update,method,metric,value\n"


# --- update descriptors and CSV (bench.hpp:22-64) ------------------------------------

def parse_update(text: str) -> RankOneUpdate:
    """"selfloop:i:w" or "edge:i:j:w" (bench.hpp:26-42)."""
    parts = text.split(":")
    try:
        if len(parts) == 3 and parts[0] == "selfloop":
            return RankOneUpdate.self_loop(_stoul(parts[1]), _stod(parts[2]))
        if len(parts) == 4 and parts[0] == "edge":
            return RankOneUpdate.edge_delta(_stoul(parts[1]), _stoul(parts[2]), _stod(parts[3]))
    except (ValueError, N.InvalidArgument):
        pass
    raise N.InvalidArgument(f"bad update descriptor '{text}' (want selfloop:i:w or edge:i:j:w)")


def _stoul(s: str) -> int:
    """std::stoul: leading whitespace, then the longest digit prefix."""
    m = re.match(r"\s*\+?(\d+)", s)
    if not m:
        raise ValueError(s)
    return int(m.group(1))


def _stod(s: str) -> float:
    """std::stod: the longest floating-point prefix."""
    m = re.match(r"\s*([+-]?(\d+\.?\d*|\.\d+)([eE][+-]?\d+)?|[+-]?(inf|infinity|nan))", s, re.IGNORECASE)
    if not m:
        raise ValueError(s)
    return float(m.group(1))


def format_update(u: RankOneUpdate) -> str:
    """bench.hpp:44-51 (an ostream prints doubles like %g)."""
    if u.kind == 0:
        return f"selfloop:{u.node_i}:{u.rho:g}"
    return f"edge:{u.node_i}:{u.node_j}:{u.rho:g}"


def csv_row(mode: str, size: int, update: str, method: str, metric: str, value: float) -> str:
    return f"{mode},{size},{update},{method},{metric},{value:.6e}\n"


# --- helpers ----------------------------------------------------------------------

def _torch():
    import torch

    if not torch.cuda.is_available():
        raise N.RuntimeFailure("the CLI runs its transforms on a CUDA device; none is visible")
    return torch


def _snr_rows(ref: np.ndarray, test: np.ndarray) -> np.ndarray:
    """signal.hpp:57-70 per row, +inf -> 320 dB as bench.hpp:189 keeps it."""
    num = np.sum(ref * ref, axis=1)
    den = np.sum((ref - test) ** 2, axis=1)
    with np.errstate(divide="ignore"):
        v = 10.0 * np.log10(num / den)
    v[den == 0.0] = 320.0
    return v


def _timed_ms(torch, fn) -> float:
    """Best of two CUDA-event-timed calls (after one warm call)."""
    fn()
    torch.cuda.synchronize()
    best = math.inf
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


class Config:
    def __init__(self, sizes: Sequence[int] = (8, 16, 32, 64, 128, 256), trials: int = 1000,
                 updates: Sequence[str] = ("selfloop:1:1.5", "edge:2:3:1.5", "edge:3:5:1.5"), epsilon: float = 1e-12,
                 seed: int = 1, cp: int = 0, threshold: float = -1.0, ar_coefficient: float = 0.99):
        self.sizes, self.trials, self.updates = list(sizes), int(trials), list(updates)
        self.epsilon, self.seed, self.cp, self.threshold = epsilon, int(seed), int(cp), threshold
        self.ar_coefficient = ar_coefficient

    def validate(self):
        """bench.hpp:79-84."""
        if not self.sizes:
            raise N.InvalidArgument("BenchConfig: no sizes")
        if any(n < 2 for n in self.sizes):
            raise N.InvalidArgument("BenchConfig: sizes must be >= 2")
        if self.trials < 1:
            raise N.InvalidArgument("BenchConfig: trials must be >= 1")


# --- runners (bench.hpp:176-372) -----------------------------------------------------

def run_accuracy(cfg: Config) -> str:
    """Mean SNR of the structured route against the dense product per cell."""
    cfg.validate()
    torch = _torch()
    out = [CSV_HEADER]
    for n in cfg.sizes:
        for k, us in enumerate(cfg.updates):
            plan = DctPlusPlan(n, parse_update(us), cfg.epsilon)
            s = fill_signals(mix_seed(cfg.seed, n, k), DIST_AR, n, cfg.trials, cfg.ar_coefficient)
            x = torch.as_tensor(s, device="cuda")
            fast = plan.forward(x).cpu().numpy()
            oracle = plan.forward_nmvp(x).cpu().numpy()
            out.append(csv_row("accuracy", n, us, "fastdctplus", "mean_snr_db", float(np.mean(_snr_rows(oracle, fast)))))
    return "".join(out)


def run_runtime(cfg: Config) -> str:
    """Per-signal batched runtimes of dct / fastdctplus / nmvp and setup."""
    import time

    cfg.validate()
    torch = _torch()
    DctPlusPlan(16, RankOneUpdate.self_loop(1, 1.0), cfg.epsilon)  # device and library init, untimed
    out = [CSV_HEADER]
    for n in cfg.sizes:
        for k, us in enumerate(cfg.updates):
            u = parse_update(us)
            t0 = time.perf_counter()
            DctPlusPlan(n, u, cfg.epsilon)
            setup_ns = (time.perf_counter() - t0) * 1e9
            plan = DctPlusPlan(n, u, cfg.epsilon)
            s = fill_signals(mix_seed(cfg.seed, n, k), DIST_AR, n, cfg.trials, cfg.ar_coefficient)
            x = torch.as_tensor(s, device="cuda")
            y = torch.empty_like(x)
            per = 1e6 / cfg.trials
            dct_ns = _timed_ms(torch, lambda: dct2(x)) * per
            fast_ns = _timed_ms(torch, lambda: plan.forward(x, sync=False, out=y)) * per
            nmvp_ns = _timed_ms(torch, lambda: plan.forward_nmvp(x, sync=False, out=y)) * per
            plan.sync_check()
            out += [csv_row("runtime", n, us, "dct", "mean_ns", dct_ns),
                    csv_row("runtime", n, us, "fastdctplus", "mean_ns", fast_ns),
                    csv_row("runtime", n, us, "nmvp", "mean_ns", nmvp_ns),
                    csv_row("runtime", n, us, "fastdctplus", "setup_ns", setup_ns),
                    csv_row("runtime", n, us, "dct", "ratio_to_dct", 1.0),
                    csv_row("runtime", n, us, "fastdctplus", "ratio_to_dct", fast_ns / dct_ns),
                    csv_row("runtime", n, us, "nmvp", "ratio_to_dct", nmvp_ns / dct_ns)]
    return "".join(out)


def measure_prune_cell(n: int, cp: int, threshold: float, epsilon: float, trials: int, seed: int,
                       ar_coefficient: float = 0.99) -> dict:
    """bench.hpp:232-336 on the GPU: the k = 3 ensemble (DCT, self-loop 1.5
    at node 1, edge 1.5 on (2,3)) at keep-count cp."""
    torch = _torch()
    ups = [RankOneUpdate.self_loop(1, 1.5), RankOneUpdate.edge_delta(2, 3, 1.5)]
    plan = PrunedEnsemblePlan(n, ups, cp, threshold, epsilon)
    members = [plan.member(r) for r in range(1, plan.ensemble_size())]
    pool = min(trials, 512)
    s = fill_signals(seed, DIST_AR, n, pool, ar_coefficient)
    x = torch.as_tensor(s, device="cuda")
    ys = [torch.empty_like(x) for _ in members]
    use_fast = []
    for m, y in zip(members, ys):
        f = _timed_ms(torch, lambda: m.forward(x, sync=False, out=y))
        d = _timed_ms(torch, lambda: m.forward_nmvp(x, sync=False, out=y))
        use_fast.append(f < d)

    def direct():
        outs = [dct2(x)]
        for m, y, fast in zip(members, ys, use_fast):
            (m.forward if fast else m.forward_nmvp)(x, sync=False, out=y)
            outs.append(y)
        return outs

    direct_ms = _timed_ms(torch, direct)
    yall = torch.empty((pool, plan.ensemble_size(), n), dtype=x.dtype, device=x.device)
    pruned_ms = _timed_ms(torch, lambda: plan.forward_all_batch(x, sync=False, out=yall))
    d = np.stack([o.cpu().numpy() for o in direct()], axis=1)            # (pool, K+1, n)
    a, _, pr = plan.forward_all_batch(x, with_bounds=True)
    a, pr = a.cpu().numpy(), pr.cpu().numpy()
    mse = np.mean((d - a) ** 2, axis=2)                                   # (pool, K+1)
    peak = float(np.max(np.abs(d)))
    mean_mse = float(np.mean(mse))
    l1d, l1a = np.sum(np.abs(d), axis=2), np.sum(np.abs(a), axis=2)
    agree = np.argmin(l1d, axis=1) == np.argmin(l1a, axis=1)             # argmin: ties to the lower index
    return {"direct_ns": direct_ms * 1e6 / pool, "pruned_ns": pruned_ms * 1e6 / pool,
            "speedup": direct_ms / pruned_ms, "mean_mse": mean_mse, "max_mse": float(np.max(mse)),
            "psnr_db": 320.0 if mean_mse == 0.0 else 10.0 * math.log10(peak * peak / mean_mse),
            "selection_agreement": float(np.mean(agree)), "prune_rate": float(np.mean(pr != 0))}


def run_prune(cfg: Config) -> str:
    cfg.validate()
    ens = "selfloop:1:1.5+edge:2:3:1.5"
    out = [CSV_HEADER]
    for n in cfg.sizes:
        thr = cfg.threshold if cfg.threshold >= 0.0 else calibrate_prune_threshold(n, cfg.ar_coefficient, 0.7, 512,
                                                                                   cfg.seed)
        cps = [min(cfg.cp, n)] if cfg.cp > 0 else [max(1, i * n // 8) for i in range(1, 9)]
        for cp in cps:
            r = measure_prune_cell(n, cp, thr, cfg.epsilon, cfg.trials, mix_seed(cfg.seed, n, cp), cfg.ar_coefficient)
            method = f"pruned_cp{cp}"
            out.append(csv_row("prune", n, ens, "direct", "mean_ns", r["direct_ns"]))
            for metric in ("mean_ns", "speedup", "mean_mse", "max_mse", "psnr_db", "selection_agreement",
                           "prune_rate"):
                out.append(csv_row("prune", n, ens, method, metric, r["pruned_ns"] if metric == "mean_ns" else r[metric]))
            out.append(csv_row("prune", n, ens, method, "threshold", thr))
    return "".join(out)


def write_signal(values) -> str:
    return " ".join(f"{v:.17g}" for v in values) + "\n"


# --- command line (fastdctplus.cpp) ---------------------------------------------------

def main(argv: List[str] = None) -> int:
    ap = argparse.ArgumentParser(prog="fastdctplus",
                                 description="Fast graph Fourier transforms for rank-one updates of the path graph")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name, hlp in (("accuracy", "mean SNR of Fast DCT+ vs the dense product"),
                      ("runtime", "per-signal runtimes and DCT-normalized ratios"),
                      ("prune", "pruned multi-transform ensemble experiment")):
        p = sub.add_parser(name, help=hlp)
        p.add_argument("--sizes", default="8,16,32,64,128,256")
        p.add_argument("--trials", type=int, default=1000)
        p.add_argument("--update", action="append", default=[])
        p.add_argument("--eps", type=float, default=1e-12)
        p.add_argument("--seed", type=int, default=1)
        p.add_argument("--cp", type=int, default=0)
        p.add_argument("--threshold", type=float, default=-1.0)
        p.add_argument("--out", default="")
    tr = sub.add_parser("transform", help="transform one signal (stdin or --in)")
    tr.add_argument("--update", default="")
    tr.add_argument("--graph", default="")
    tr.add_argument("--in", dest="inp", default="")
    tr.add_argument("--eps", type=float, default=1e-12)
    tr.add_argument("--inverse", action="store_true")
    a = ap.parse_args(argv)
    try:
        if a.cmd == "transform":
            text = open(a.inp).read() if a.inp else sys.stdin.read()
            s = np.array([float(v) for v in text.split()])
            if s.size < 2:
                raise N.RuntimeFailure("signal needs at least 2 samples")
            if a.graph:
                raise N.RuntimeFailure("--graph (dense general-graph GFT) is not part of this library")
            if not a.update:
                raise N.RuntimeFailure("transform needs --update or --graph")
            plan = DctPlusPlan(s.size, parse_update(a.update), a.eps)
            sys.stdout.write(write_signal(plan.inverse(s) if a.inverse else plan.forward(s)))
            return 0
        cfg = Config(sizes=[int(v) for v in a.sizes.split(",") if v], trials=a.trials,
                     updates=a.update or ("selfloop:1:1.5", "edge:2:3:1.5", "edge:3:5:1.5"), epsilon=a.eps,
                     seed=a.seed, cp=a.cp, threshold=a.threshold)
        text = {"accuracy": run_accuracy, "runtime": run_runtime, "prune": run_prune}[a.cmd](cfg)
        if not a.out or a.out == "-":
            sys.stdout.write(text)
        else:
            with open(a.out, "w") as f:
                f.write(text)
        return 0
    except Exception as e:  # noqa: BLE001 — the reference prints every std::exception this way
        sys.stderr.write(f"error: {e}\n")
        return 1


if __name__ == "__main__":
    sys.exit(main())
