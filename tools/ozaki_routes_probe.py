"""Development probe: every route that uses the int8 tcgen05 (Ozaki) products
(C3 folded forward / inverse fp64, C5 dense, the X6 rank-k chain) against the
same route on the DMMA pipe (DCTP_OZAKI=0), plus kernel times from the
library's per-launch CUDA events."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_08970_b200 as P  # noqa: E402
from paper_2409_08970_b200.configs import WORKLOADS, make_plan  # noqa: E402


def timed(fn, reps=10):
    P.profile_reset()
    P.profile_enable(True)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    P.profile_enable(False)
    return {k: round(v[1] / v[0], 4) for k, v in P.profile_summary().items()}


def err(a, b):
    return ((a - b).abs().amax(dim=1) / b.abs().amax(dim=1)).max().item()


for cid, ops in ((3, ("fwd", "inv")), (5, ("fwd", "inv")), (6, ("fwd",))):
    cfg = WORKLOADS[cid]
    plan = make_plan(cfg)
    x = torch.as_tensor(P.fill_signals(cfg.seed, cfg.dist, cfg.n, cfg.batch, cfg.r), device="cuda")
    for op in ops:
        fn = plan.forward if op == "fwd" else plan.inverse
        res = {}
        for mode in ("0", "1"):
            os.environ["DCTP_OZAKI"] = mode
            y = fn(x)
            out = torch.empty_like(x)
            t = timed(lambda: fn(x, sync=False, out=out))
            res[mode] = (y, t)
        print(f"C{cid} {op}: ozaki vs dmma {err(res['1'][0], res['0'][0]):.3e}  dmma {res['0'][1]}  "
              f"ozaki {res['1'][1]}", flush=True)
    del plan
    torch.cuda.empty_cache()
