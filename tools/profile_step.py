"""Run one BASELINE workload's step `--reps` times (device-resident inputs, as
in bench.py) — the command the ncu captures under profiles/ wrap.
usage: python tools/profile_step.py C5 [--reps 4] [--env K=V ...]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("key")
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--batch", type=int, default=0, help="override the batch (0: the BASELINE batch)")
args = ap.parse_args()

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2409_08970_b200 as P  # noqa: E402
from paper_2409_08970_b200.configs import WORKLOADS, make_plan  # noqa: E402

cfg = bench.CONFIGS[args.key]
plan = make_plan(WORKLOADS[cfg["cid"]])
batch = args.batch or cfg["batch"]
dtype = torch.float32 if cfg["dtype"] == "f32" else torch.float64
x = torch.as_tensor(P.fill_signals(P.mix_seed(2409, cfg["n"], cfg["cid"]), cfg["dist"], cfg["n"], batch, cfg["r"]),
                    device="cuda").to(dtype)
op = cfg["op"]
if op == "inverse":
    x = plan.forward(x)
for _ in range(args.reps):
    if op == "forward_all":
        y = plan.forward_all_batch(x, sync=False)
    elif op == "inverse":
        y = plan.inverse(x, sync=False)
    else:
        y = plan.forward(x, sync=False)
torch.cuda.synchronize()
print("ok", args.key, tuple(y.shape))
