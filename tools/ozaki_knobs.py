"""Development probe: a workload's kernel times (CID, default 5 = C5) under
environment knobs, one subprocess per setting.  Usage: python tools/ozaki_knobs.py 'A=1 B=2' ''"""
import json
import os
import subprocess
import sys

CHILD = r'''
import os, sys, json, torch
sys.path.insert(0, os.getcwd())
import paper_2409_08970_b200 as P
from paper_2409_08970_b200.configs import WORKLOADS, make_plan
cfg = WORKLOADS[int(os.environ.get("CID", "5"))]
if os.environ.get("BATCH"):
    import dataclasses
    cfg = dataclasses.replace(cfg, batch=int(os.environ["BATCH"]))
plan = make_plan(cfg)
x = torch.as_tensor(P.fill_signals(cfg.seed, cfg.dist, cfg.n, cfg.batch, cfg.r), device="cuda")
if cfg.progressive:
    x = x.float()
    out = torch.empty((x.shape[0], 17, cfg.n), dtype=x.dtype, device=x.device)
    fn = plan.forward_all_batch
else:
    if os.environ.get("DTYPE") == "f32":
        x = x.float()
    if os.environ.get("OP") == "inv":
        x = plan.forward(x)
    out = torch.empty_like(x)
    fn = plan.inverse if os.environ.get("OP") == "inv" else plan.forward
for _ in range(3):
    fn(x, sync=False, out=out)
torch.cuda.synchronize()
P.profile_reset(); P.profile_enable(True)
for _ in range(10):
    fn(x, sync=False, out=out)
torch.cuda.synchronize(); P.profile_enable(False)
if os.environ.get("SAVE"):
    import numpy as np
    np.save(os.environ["SAVE"], out.double().cpu().numpy())
print(json.dumps({k: round(v[1] / v[0], 4) for k, v in P.profile_summary().items()}))
'''
first = None
for i, setting in enumerate(sys.argv[1:]):
    env = dict(os.environ)
    for kv in setting.split():
        k, v = kv.split("=")
        env[k] = v
    env["SAVE"] = f"/tmp/ozaki_knobs_{i}.npy"
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
    gap = ""
    if r.returncode == 0:  # max |y - y_first| / max |y_first| against the first setting's output
        import numpy as np
        y = np.load(env["SAVE"])
        if first is None:
            first = y
        elif y.shape == first.shape:
            gap = f" gap={np.abs(y - first).max() / np.abs(first).max():.2e}"
    print(repr(setting), (r.stdout.strip() or r.stderr[-2000:]) + gap, flush=True)
