"""DCTP_DEBUG_MODE bit 4: phase accounting of the lock-step fused kernel (thread 0 of each CTA)."""
import ctypes, os, sys
from pathlib import Path
os.environ["DCTP_DEBUG_MODE"] = str(4 | int(os.environ.get("DCTP_DEBUG_MODE", "0")))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2409_08970_b200 as P
from paper_2409_08970_b200 import _native
from paper_2409_08970_b200.configs import WORKLOADS, make_plan
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = WORKLOADS[cid]
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
names = ["wait_load", "phaseA_dct", "sync1_wait", "phaseB_dmma", "sync2_wait", "loop_top", "t0_store_claim"]
tot = sum(buf[:6])
for i, nm in enumerate(names):  # slots 0-5: thread 32's loop (sums to its total); 6: thread 0's duty
    print(f"{nm:12s} {buf[i] / tiles:8.0f} cycles/tile {100 * buf[i] / max(tot, 1):5.1f}%")
print(f"total {tot / 148 / 1.965e3:.1f} us per CTA at 1965 MHz")
