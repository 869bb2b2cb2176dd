"""Small-batch end-to-end paths (C1: 4096 x 64 fp64): the pipelined host
entry against a zero-copy call where the fused kernel's TMA copies read and
write the pinned host buffers directly over PCIe.

usage (GPU box): python tools/small_e2e_probe.py [config]
"""
import ctypes as C
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2409_08970_b200._native import check, lib  # noqa: E402
from paper_2409_08970_b200.configs import WORKLOADS, make_plan  # noqa: E402


def main():
    cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    cfg = WORKLOADS[cid]
    plan = make_plan(cfg)
    res = {}
    for batch in (1024, 4096, 16384, 65536):
        shape = (batch, cfg.n)
        h_in = torch.randn(shape, dtype=torch.float64).pin_memory()
        h_out = torch.empty(shape, dtype=torch.float64).pin_memory()
        s = torch.cuda.current_stream()
        sp = C.c_void_p(s.cuda_stream)

        def host_entry():
            check(lib.dctp_forward_host_f64(plan._h, C.c_void_p(h_in.data_ptr()), C.c_void_p(h_out.data_ptr()),
                                            batch))

        def zero_copy():
            check(lib.dctp_forward_f64(plan._h, C.c_void_p(h_in.data_ptr()), C.c_void_p(h_out.data_ptr()), batch,
                                       sp))
            check(lib.dctp_plan_sync_check(plan._h, sp))

        d_in, d_out = h_in.cuda(), torch.empty(shape, dtype=torch.float64, device="cuda")

        def one_stream():
            d_in.copy_(h_in, non_blocking=True)
            check(lib.dctp_forward_f64(plan._h, C.c_void_p(d_in.data_ptr()), C.c_void_p(d_out.data_ptr()), batch,
                                       sp))
            h_out.copy_(d_out, non_blocking=True)
            check(lib.dctp_plan_sync_check(plan._h, sp))

        for name, fn in (("host_entry", host_entry), ("zero_copy", zero_copy), ("one_stream", one_stream)):
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            t = time.perf_counter()
            reps = 50
            for _ in range(reps):
                fn()
            dt = (time.perf_counter() - t) / reps
            res[f"{name} batch={batch}"] = {"us": dt * 1e6, "samples_per_s": batch * cfg.n / dt}
        ref = h_out.clone()
        host_entry()
        zero_copy()
        res[f"zero_copy matches host_entry batch={batch}"] = bool(torch.equal(ref, h_out))
    for k, v in res.items():
        print(cid, k, json.dumps(v))


if __name__ == "__main__":
    main()
