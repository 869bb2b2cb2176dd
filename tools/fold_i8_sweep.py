"""C2-shape plan (n = 256, edge (128, 129), -0.7): the grouped int8 route
(DCTP_FOLD_I8=1) against the fused DMMA kernel (DCTP_FOLD_I8=0) — GPU time per
forward (CUDA events, 20 applies) at several batches and the max per-signal
relative difference between the two routes.  Each route runs in its own
process (the knob is read per call, the plan is shared within a process).
usage (GPU box): python tools/fold_i8_sweep.py"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CODE = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_2409_08970_b200 as P
plan = P.DctPlusPlan(256, P.RankOneUpdate.edge_delta(128, 129, -0.7), 1e-12)
res = {}
for b in (1024, 4096, 8192, 16384, 32768, 65536):
    x = torch.as_tensor(P.fill_signals(P.mix_seed(2409, 256, 2), P.DIST_AR, 256, b, 0.95), device="cuda")
    y = torch.empty_like(x)
    for _ in range(3): plan.forward(x, sync=False, out=y)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): plan.forward(x, sync=False, out=y)
    e.record(); e.synchronize()
    np.save("%s_%%d.npy" %% b, y.cpu().numpy())
    res[b] = a.elapsed_time(e) / 20
print(json.dumps(res))
"""
out = {}
for mode in ("0", "1"):
    tag = f"/tmp/fold_i8_{mode}"
    r = subprocess.run([sys.executable, "-c", CODE % (str(ROOT), tag)], env=dict(os.environ, DCTP_FOLD_I8=mode),
                       capture_output=True, text=True)
    out[mode] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-500:]
import numpy as np  # noqa: E402
for b in (1024, 4096, 8192, 16384, 32768, 65536):
    y0, y1 = np.load(f"/tmp/fold_i8_0_{b}.npy"), np.load(f"/tmp/fold_i8_1_{b}.npy")
    err = float(np.max(np.max(np.abs(y1 - y0), axis=1) / np.max(np.abs(y0), axis=1)))
    print(json.dumps({"batch": b, "fused_ms": out["0"][str(b)], "fold_i8_ms": out["1"][str(b)], "max_rel_diff": err}))
