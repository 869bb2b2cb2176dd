"""Per-signal latency: the drop-in C++ DctPlusPlan::forward(s, ws) (one host
vector per call, tools/latency.cpp) against the reference's own per-signal
forward on one host thread (oracle/_ref, the loop of bench.hpp:139-169).
Writes JSON to argv[1].  ORACLE USE: the reference leg only (test tooling)."""
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
LIB = ROOT / "paper_2409_08970_b200" / "lib"
EXE = ROOT / "paper_2409_08970_b200" / "build" / "latency"
subprocess.run(["g++", "-std=c++17", "-O2", "-I", str(ROOT / "include"), "-I", "/usr/local/cuda/include",
                str(ROOT / "tools" / "latency.cpp"), "-o", str(EXE), "-L", str(LIB), "-ldctplus_b200",
                f"-Wl,-rpath,{LIB}", "-L", "/usr/local/cuda/lib64", "-lcudart"], check=True)
gpu = [json.loads(l) for l in subprocess.run([str(EXE)], capture_output=True, text=True, check=True).stdout.splitlines()]

from oracle import checkers as O  # noqa: E402

ref = O.Reference()
cases = [(64, O.Update(0, 0.5, 1)), (256, O.Update(1, -0.7, 128, 129)), (1024, O.Update(1, 1.0, 1, 1024))]
out = []
for g, (n, u) in zip(gpu, cases):
    plan = ref.plan(n, u)
    rows = max(64, int(2e5 // n))
    s = np.random.default_rng(1).standard_normal((rows, n))
    plan.forward(s[:16], threads=1)
    t = time.perf_counter()
    plan.forward(s, threads=1)
    per = (time.perf_counter() - t) / rows * 1e6
    out.append({**g, "reference_us_per_signal_1thread": round(per, 2),
                "gpu_over_reference": round(g["median_us"] / per, 2)})
res = {"what": "median latency of one DctPlusPlan::forward(s, ws) call (host vector in, host vector out) through "
               "the C++ mirror, against the reference's per-signal forward on one host thread",
       "cases": out}
Path(sys.argv[1]).write_text(json.dumps(res, indent=1))
print(json.dumps(res, indent=1))
