"""DCTP_DEBUG_MODE bit 4: per-phase cycle accounting of the fused kernel's producer."""
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
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
_native.lib.dctp_debug_timers(buf)
e0.record(); plan.forward(x, sync=False, out=y); e1.record()
torch.cuda.synchronize()
_native.lib.dctp_debug_timers(buf)
print(f"kernel {e0.elapsed_time(e1)*1e3:.1f} us; producer-warp total {buf[7] / (148 * 8):.0f} cycles "
      f"(= {buf[7] / (148 * 8) / 1.965e3:.1f} us at 1965 MHz), loop sum {sum(buf[:7]) / (148 * 8):.0f} cycles")
print(f"globaltimer: first CTA entry -> last exit {(buf[9] - buf[8]) / 1e3:.1f} us; last CTA entry at +{(buf[10] - buf[8]) / 1e3:.1f} us;"
      f" first exit at +{(buf[11] - buf[8]) / 1e3:.1f} us")
names = ["tail", "wait_xfull", "pass0", "fft_rest", "split", "wait_free", "gather"]
tot = sum(buf[:7])
tiles = (w.batch + 15) // 16
nw = 8
for i, nm in enumerate(names):
    print(f"{nm:12s} {buf[i] / tiles / nw:10.0f} cycles/tile/warp  {100 * buf[i] / max(tot, 1):5.1f}%")
