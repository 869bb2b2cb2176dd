"""Probe the host<->device path of the e2e number: raw pinned copy bandwidth
(H2D, D2H, both at once) and the host entry point at several chunk sizes.

usage (GPU box): python tools/e2e_probe.py
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def copy_bw():
    nbytes = 128 << 20
    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}

    def timeit(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def h2d():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        s1.synchronize()

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        s2.synchronize()

    def both():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        s1.synchronize()
        s2.synchronize()

    for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
        ms = timeit(fn)
        res[name] = {"ms": ms, "GBps_each": nbytes / ms / 1e6}
    return res


def host_entry(chunk_mb, slots=3, streamed=1, stream_kb=2048, min_mb=2, wl=2, floor=256):
    code = r"""
import time, numpy as np, torch, json
import paper_2409_08970_b200 as P
from paper_2409_08970_b200.configs import WORKLOADS, make_plan
cfg = WORKLOADS[WL]
plan = make_plan(cfg)
x = torch.randn(cfg.batch, cfg.n, dtype=torch.float64).pin_memory().numpy()
y = torch.empty(cfg.batch, cfg.n, dtype=torch.float64).pin_memory().numpy()
import ctypes as C
from paper_2409_08970_b200._native import check, lib
def call():
    check(lib.dctp_forward_host_f64(plan._h, C.c_void_p(x.ctypes.data), C.c_void_p(y.ctypes.data), cfg.batch))
for _ in range(3): call()
torch.cuda.synchronize()
t = time.perf_counter(); R = 10
for _ in range(R): call()
ms = (time.perf_counter() - t) / R * 1e3
print(json.dumps({"ms": ms}))
"""
    env = dict(os.environ, DCTP_HOST_CHUNK_MB=str(chunk_mb), DCTP_HOST_SLOTS=str(slots), DCTP_HOST_STREAMED=str(streamed),
               DCTP_STREAM_CHUNK_KB=str(stream_kb), DCTP_HOST_CHUNK_MIN_MB=str(min_mb), DCTP_HOST_MIN_ROWS=str(floor))
    out = subprocess.run([sys.executable, "-c", code.replace("WL", str(wl))], env=env, capture_output=True, text=True,
                         cwd=ROOT)
    try:
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:
        return {"error": out.stderr[-400:]}


if __name__ == "__main__":
    print(json.dumps({"copy_bw": copy_bw()}))
    wl = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    for mb, mn, slots, floor in ((16, 2, 3, 256), (16, 4, 4, 64), (16, 4, 6, 64), (16, 8, 6, 128), (16, 2, 6, 32),
                                 (32, 4, 6, 64), (16, 16, 6, 256), (8, 4, 6, 64)):
        print(json.dumps({"wl": wl, "staged_chunk_mb": mb, "min_mb": mn, "slots": slots, "floor": floor,
                          **host_entry(mb, slots, 0, min_mb=mn, wl=wl, floor=floor)}))
