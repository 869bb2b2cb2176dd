"""Does a concurrent PCIe copy slow the fused kernel?  Per-launch time of the
C2 kernel on 4096-row chunks, alone and while a 1 GB H2D copy runs."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2409_08970_b200._native import check, lib  # noqa: E402
from paper_2409_08970_b200.configs import WORKLOADS, make_plan  # noqa: E402

cfg = WORKLOADS[2]
plan = make_plan(cfg)
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
a = torch.randn(rows, cfg.n, dtype=torch.float64, device="cuda")
b = torch.empty_like(a)
hbig = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
dbig = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
s, sc = torch.cuda.Stream(), torch.cuda.Stream()
sp = C.c_void_p(s.cuda_stream)


def run(reps, gap_sync):
    evs = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        check(lib.dctp_forward_f64(plan._h, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), rows, sp))
        e1.record(s)
        evs.append((e0, e1))
        if gap_sync:
            s.synchronize()
    torch.cuda.synchronize()
    t = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in evs)
    return {"median_us": t[len(t) // 2], "min_us": t[0], "max_us": t[-1]}


res = {"rows": rows}
run(5, False)
res["alone_back_to_back"] = run(50, False)
res["alone_synced_each"] = run(50, True)
with torch.cuda.stream(sc):
    dbig.copy_(hbig, non_blocking=True)
res["during_h2d_back_to_back"] = run(30, False)
torch.cuda.synchronize()
with torch.cuda.stream(sc):
    dbig.copy_(hbig, non_blocking=True)
res["during_h2d_synced_each"] = run(30, True)
torch.cuda.synchronize()
print(json.dumps(res))
