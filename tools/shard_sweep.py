"""Per-GPU time of C5's forward at the shard sizes of the 1/2/4/8-GPU strong-
scaling run (2048 / G rows), CUDA events over 20 back-to-back applies on one
GPU — what each rank of `bench.py --gpus G` times (inputs resident).
usage (GPU box): python tools/shard_sweep.py"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2409_08970_b200 as P  # noqa: E402
from paper_2409_08970_b200.configs import WORKLOADS, make_plan  # noqa: E402

cfg = WORKLOADS[5]
plan = make_plan(cfg)
x_all = torch.as_tensor(P.fill_signals(P.mix_seed(2409, cfg.n, 5), cfg.dist, cfg.n, cfg.batch, cfg.r), device="cuda")
for g in (1, 2, 4, 8):
    rows = cfg.batch // g
    x = x_all[:rows].contiguous()
    y = torch.empty_like(x)
    for _ in range(3):
        plan.forward(x, sync=False, out=y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        plan.forward(x, sync=False, out=y)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 20
    print(json.dumps({"gpus": g, "rows_per_gpu": rows, "ms": round(ms, 4),
                      "ideal_ms": None, "samples_per_s_job": cfg.batch * cfg.n / (ms * 1e-3)}))
