"""Where does the e2e time go?  Time the C2 fused kernel with each operand in
device memory or in pinned host memory (read / written over PCIe by the
kernel's TMA bulk copies), and a plain torch 3-stream staged pipeline.

usage (GPU box): python tools/zc_probe.py
"""
import ctypes as C
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2409_08970_b200._native import check, lib  # noqa: E402
from paper_2409_08970_b200.configs import WORKLOADS, make_plan  # noqa: E402


def main():
    cfg = WORKLOADS[2]
    plan = make_plan(cfg)
    shape = (cfg.batch, cfg.n)
    h_in = torch.randn(shape, dtype=torch.float64).pin_memory()
    h_out = torch.empty(shape, dtype=torch.float64).pin_memory()
    d_in = h_in.cuda()
    d_out = torch.empty(shape, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)

    def timed(fn, reps=10):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    res = {}
    for name, a, b in (("dev->dev", d_in, d_out), ("host->dev", h_in, d_out), ("dev->host", d_in, h_out),
                       ("host->host", h_in, h_out)):
        res[name] = timed(lambda: check(lib.dctp_forward_f64(plan._h, C.c_void_p(a.data_ptr()),
                                                             C.c_void_p(b.data_ptr()), cfg.batch, sp)))
    # torch staged pipeline: copy-in / compute / copy-out streams, 8 MB chunks
    rows = 4096
    sin, scomp, sout = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    slots = 3
    bin_ = [torch.empty((rows, cfg.n), dtype=torch.float64, device="cuda") for _ in range(slots)]
    bout = [torch.empty((rows, cfg.n), dtype=torch.float64, device="cuda") for _ in range(slots)]
    ev_l = [torch.cuda.Event() for _ in range(slots)]
    ev_c = [torch.cuda.Event() for _ in range(slots)]
    ev_d = [torch.cuda.Event() for _ in range(slots)]

    def staged(kernel="ours"):
        for c, r0 in enumerate(range(0, cfg.batch, rows)):
            k = c % slots
            if c >= slots:
                sin.wait_event(ev_c[k])
            with torch.cuda.stream(sin):
                bin_[k].copy_(h_in[r0:r0 + rows], non_blocking=True)
                ev_l[k].record(sin)
            scomp.wait_event(ev_l[k])
            if c >= slots:
                scomp.wait_event(ev_d[k])
            if kernel == "torch_copy":
                with torch.cuda.stream(scomp):
                    bout[k].copy_(bin_[k])
            elif kernel == "ours":
                check(lib.dctp_forward_f64(plan._h, C.c_void_p(bin_[k].data_ptr()), C.c_void_p(bout[k].data_ptr()),
                                           rows, C.c_void_p(scomp.cuda_stream)))
            ev_c[k].record(scomp)
            sout.wait_event(ev_c[k])
            with torch.cuda.stream(sout):
                h_out[r0:r0 + rows].copy_(bout[k], non_blocking=True)
                ev_d[k].record(sout)
        torch.cuda.synchronize()

    import time
    for kern in ("ours", "torch_copy", "none"):
        staged(kern)
        t = time.perf_counter()
        for _ in range(10):
            staged(kern)
        res[f"torch staged 8MB kernel={kern}"] = (time.perf_counter() - t) / 10 * 1e3
    print(json.dumps(res, indent=1))

    # timeline of one staged run (events on each stream, ms from the start)
    for kern in ("ours", "none"):
        E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        base = E()
        torch.cuda.synchronize()
        base.record(sin)
        marks = []
        for c, r0 in enumerate(range(0, cfg.batch, rows)):
            k = c % slots
            m = [E() for _ in range(6)]
            if c >= slots:
                sin.wait_event(ev_c[k])
            m[0].record(sin)
            with torch.cuda.stream(sin):
                bin_[k].copy_(h_in[r0:r0 + rows], non_blocking=True)
                ev_l[k].record(sin)
            m[1].record(sin)
            scomp.wait_event(ev_l[k])
            if c >= slots:
                scomp.wait_event(ev_d[k])
            m[2].record(scomp)
            if kern == "ours":
                check(lib.dctp_forward_f64(plan._h, C.c_void_p(bin_[k].data_ptr()), C.c_void_p(bout[k].data_ptr()),
                                           rows, C.c_void_p(scomp.cuda_stream)))
            m[3].record(scomp)
            ev_c[k].record(scomp)
            sout.wait_event(ev_c[k])
            m[4].record(sout)
            with torch.cuda.stream(sout):
                h_out[r0:r0 + rows].copy_(bout[k], non_blocking=True)
                ev_d[k].record(sout)
            m[5].record(sout)
            marks.append(m)
        torch.cuda.synchronize()
        print(kern)
        for c, m in enumerate(marks):
            print(c, " ".join(f"{base.elapsed_time(e):7.3f}" for e in m))


if __name__ == "__main__":
    main()
