"""Development probe: small plans (n = 64 / 128) across batch sizes, the
one-launch dense kernel (DCTP_SMALL_DENSE=1) against the fused persistent
kernel (=0); per-launch CUDA-event times, one subprocess per setting."""
import json
import os
import subprocess
import sys

CHILD = r'''
import os, sys, json, torch
sys.path.insert(0, os.getcwd())
import paper_2409_08970_b200 as P
res = {}
for n, upd in ((64, P.RankOneUpdate.self_loop(1, 0.5)), (128, P.RankOneUpdate.self_loop(1, 0.7))):
    plan = P.DctPlusPlan(n, upd, 1e-12)
    for b in (1, 64, 1024, 4096, 16384, 65536):
        x = torch.as_tensor(P.fill_signals(3, 0, n, b), device="cuda")
        y = torch.empty_like(x)
        for _ in range(5):
            plan.forward(x, sync=False, out=y)
        torch.cuda.synchronize()
        # GPU time per forward: 20 forwards captured in a CUDA graph and
        # replayed (no host overhead between launches)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            plan.forward(x, sync=False, out=y)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(20):
                    plan.forward(x, sync=False, out=y)
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); e1.synchronize()
        res[f"n{n}_b{b}"] = round(e0.elapsed_time(e1) * 1e3 / 20, 1)
print(json.dumps(res))
'''
for setting in ("DCTP_SMALL_DENSE=1", "DCTP_SMALL_DENSE=0"):
    env = dict(os.environ)
    k, v = setting.split("=")
    env[k] = v
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
    print(setting, r.stdout.strip() or r.stderr[-2000:], flush=True)
