"""One traced streamed host-buffer forward of C2 (DCTP_STREAM_TRACE=1 prints a
per-chunk timeline: input landed / all tiles stored / output drained)."""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ.setdefault("DCTP_STREAM_TRACE", "1")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2409_08970_b200._native import check, lib  # noqa: E402
from paper_2409_08970_b200.configs import WORKLOADS, make_plan  # noqa: E402

cfg = WORKLOADS[2]
plan = make_plan(cfg)
x = torch.randn(cfg.batch, cfg.n, dtype=torch.float64).pin_memory()
y = torch.empty_like(x).pin_memory()
for _ in range(int(os.environ.get("REPS", "2"))):
    check(lib.dctp_forward_host_f64(plan._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), cfg.batch))
    print("---", file=sys.stderr)
