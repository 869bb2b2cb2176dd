"""DCTP_DEBUG_MODE bit 4: per-step cycle split of the C2 ping-pong kernel
(group 0 = warps 0-7: DMMA then DCT; group 1 = warps 8-15: DCT then DMMA)."""
import ctypes
import os
import sys
from pathlib import Path

os.environ["DCTP_DEBUG_MODE"] = "4"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2409_08970_b200 as P  # noqa: E402
from paper_2409_08970_b200 import _native  # noqa: E402
from paper_2409_08970_b200.configs import WORKLOADS, make_plan  # noqa: E402

w = WORKLOADS[2]
plan = make_plan(w)
x = torch.as_tensor(P.fill_signals(w.seed, w.dist, w.n, w.batch, w.r), device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    plan.forward(x, sync=False, out=y)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
_native.lib.dctp_debug_timers(buf)
plan.forward(x, sync=False, out=y)
torch.cuda.synchronize()
_native.lib.dctp_debug_timers(buf)
tiles = (w.batch + 15) // 16
for g, names in ((0, ("dmma", "dct", "barrier")), (3, ("dct", "dmma", "barrier"))):
    print(f"group {g // 3}: " + "  ".join(f"{nm} {buf[g + i] / tiles:7.0f}" for i, nm in enumerate(names)) + " cycles/tile")
