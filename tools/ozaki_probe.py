"""Development probe: the int8 tcgen05 (Ozaki) dense route against the DMMA
dense route and the reference's C5 goldens; kernel times from the library's
per-launch CUDA events.  Usage: python tools/ozaki_probe.py [slices]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    os.environ["DCTP_OZAKI_SLICES"] = sys.argv[1]
import paper_2409_08970_b200 as P  # noqa: E402
from oracle import checkers as O  # noqa: E402
from paper_2409_08970_b200.configs import WORKLOADS, make_plan  # noqa: E402
from tests.golden_io import load_golden  # noqa: E402


def timed(fn, reps=10):
    P.profile_reset()
    P.profile_enable(True)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    P.profile_enable(False)
    return {k: v[1] / v[0] for k, v in P.profile_summary().items()}


cfg = WORKLOADS[5]
t = time.time()
plan = make_plan(cfg)
print("plan", time.time() - t, flush=True)
g = load_golden("c5")
s = torch.as_tensor(g["signals"], device="cuda")
for mode in ("0", "1"):
    os.environ["DCTP_OZAKI"] = mode
    y = plan.forward(s).cpu().numpy()
    print("mode", mode, "golden parity", O.parity(y, g["forward"]), flush=True)

x = torch.as_tensor(P.fill_signals(cfg.seed, cfg.dist, cfg.n, cfg.batch, cfg.r), device="cuda")
os.environ["DCTP_OZAKI"] = "0"
y0 = plan.forward(x)
os.environ["DCTP_OZAKI"] = "1"
t = time.time()
y1 = plan.forward(x)
torch.cuda.synchronize()
print("first ozaki call (slices X^T)", time.time() - t)
err = ((y1 - y0).abs().amax(dim=1) / y0.abs().amax(dim=1)).max().item()
print("full batch ozaki vs dmma", err, flush=True)
for mode in ("0", "1"):
    os.environ["DCTP_OZAKI"] = mode
    out = torch.empty_like(x)
    print("mode", mode, timed(lambda: plan.forward(x, sync=False, out=out)), flush=True)
