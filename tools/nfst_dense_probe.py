"""Development probe: NFST kernel vs its materialised int8 operator at n =
1024..8192 (self-loop plans of weight 0.5 / 5.0 from n = 2048, NFST route forced with DCTP_FAST=1): time per batch (CUDA events)
and the max-norm gap between the two.  usage: python tools/nfst_dense_probe.py"""
import json
import os
import subprocess
import sys

CHILD = r'''
import os, sys, json, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2409_08970_b200 as P
n, batch, op = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
plan = P.DctPlusPlan(n, P.RankOneUpdate.self_loop(1, 0.5 if n <= 1024 else 5.0), 1e-12)
x = torch.as_tensor(P.fill_signals(11, 0, n, batch), device="cuda")
fn = plan.forward if op == "fwd" else plan.inverse
out = torch.empty_like(x)
for _ in range(3):
    fn(x, sync=False, out=out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    fn(x, sync=False, out=out)
b.record(); torch.cuda.synchronize()
np.save(sys.argv[4], out.cpu().numpy())
print(json.dumps({"route_nfst": plan.route()["nfst"], "ms": a.elapsed_time(b) / 10}))
'''
for n, batch in ((2048, 8192), (4096, 4096), (8192, 2048)):
    for op in ("fwd", "inv"):
        res = {}
        for mode in ("0", "1"):
            env = dict(os.environ, DCTP_NFST_DENSE=mode, DCTP_NFST_DENSE_MAX_N="8192", DCTP_FAST="1")
            f = f"/tmp/nfst_{n}_{op}_{mode}.npy"
            r = subprocess.run([sys.executable, "-c", CHILD, str(n), str(batch), op, f], env=env, capture_output=True,
                               text=True, timeout=900)
            res[mode] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-500:]
        import numpy as np
        try:
            y0, y1 = np.load(f"/tmp/nfst_{n}_{op}_0.npy"), np.load(f"/tmp/nfst_{n}_{op}_1.npy")
            gap = float(np.abs(y0 - y1).max() / np.abs(y0).max())
        except Exception:
            gap = None
        print(json.dumps({"n": n, "batch": batch, "op": op, "kernel": res["0"], "int8_operator": res["1"], "gap": gap}),
              flush=True)
