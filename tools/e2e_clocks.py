"""SM clocks and per-launch kernel time during the host-buffer (e2e) loop."""
import ctypes as C
import json
import os
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import pynvml  # noqa: E402
import torch  # noqa: E402

import paper_2409_08970_b200 as P  # noqa: E402
from paper_2409_08970_b200._native import check, lib  # noqa: E402
from paper_2409_08970_b200.configs import WORKLOADS, make_plan  # noqa: E402

cfg = WORKLOADS[2]
plan = make_plan(cfg)
x = torch.randn(cfg.batch, cfg.n, dtype=torch.float64).pin_memory()
y = torch.empty_like(x).pin_memory()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        time.sleep(0.005)


def call():
    check(lib.dctp_forward_host_f64(plan._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), cfg.batch))


for _ in range(3):
    call()
t = threading.Thread(target=sampler)
t.start()
P.profile_enable(True)
t0 = time.perf_counter()
R = 200
for _ in range(R):
    call()
ms = (time.perf_counter() - t0) / R * 1e3
P.profile_enable(False)
stop.set()
t.join()
prof = P.profile_summary()
samples.sort()
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("DCTP_")}, "ms_per_call": ms,
                  "sm_mhz_median": samples[len(samples) // 2], "sm_mhz_min": samples[0], "n": len(samples),
                  "kernels": {k: [v[0], v[1] / max(v[0], 1)] for k, v in prof.items()}}))
