#!/usr/bin/env python3
"""Route crossover sweep (fp64 forward): the NFST fast route (DCTP_FAST=1)
against the exact routes the plan would otherwise take (DCTP_FAST=0), on
device-resident batches of 2^24 / n signals (128 MiB in, 128 MiB out), CUDA
events over 20 launches after 3 warm-ups.  Prints one JSON line per plan;
the default DCTP_FAST_MIN_N in capi.cpp comes from these numbers.

  python tools/route_sweep.py [n ...]
"""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2409_08970_b200 as P  # noqa: E402

R = P.RankOneUpdate
CASES = {
    128: [R.self_loop(1, 0.5), R.edge_delta(64, 65, -0.7)],
    256: [R.self_loop(1, 0.5), R.edge_delta(128, 129, -0.7)],
    512: [R.self_loop(1, 1.3), R.edge_delta(256, 257, 2.0)],
    1024: [R.self_loop(1, 0.5), R.edge_delta(512, 513, 2.0)],
    2048: [R.self_loop(1, 5.0), R.edge_delta(1024, 1025, 2.0)],
}


def time_forward(plan, x, y, reps=20):
    for _ in range(3):
        plan.forward(x, out=y, sync=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        plan.forward(x, out=y, sync=False)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ns = [int(a) for a in sys.argv[1:]] or sorted(CASES)
    for n in ns:
        for u in CASES[n]:
            plan = P.DctPlusPlan(n, u, 1e-12)
            if plan.slow_path():
                continue
            batch = (1 << 24) // n
            x = torch.randn(batch, n, dtype=torch.float64, device="cuda")
            y = torch.empty_like(x)
            res = {"n": n, "update": repr(u), "batch": batch, "kept": plan.n_kept, "active": plan.n_active}
            for mode in ("0", "1"):
                os.environ["DCTP_FAST"] = mode
                P.profile_reset()
                P.profile_enable(True)
                plan.forward(x, out=y)
                P.profile_enable(False)
                kern = sorted(P.profile_summary())
                ms = time_forward(plan, x, y)
                res["fast" if mode == "1" else "exact"] = {"ms": round(ms, 4), "kernels": kern,
                                                           "samples_per_s": batch * n / ms * 1e3}
            os.environ.pop("DCTP_FAST")
            res["fast_over_exact"] = round(res["exact"]["ms"] / res["fast"]["ms"], 3)
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
