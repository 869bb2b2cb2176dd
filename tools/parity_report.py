"""Full-batch parity numbers (the values tests/test_full_batch_parity.py
asserts against): every BASELINE config, every signal, against the reference
compiled in place (oracle/_ref) on all host threads.  Writes JSON to argv[1].
ORACLE USE: test infrastructure only (the checker), never the product path."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2409_08970_b200 as P  # noqa: E402
from oracle import checkers as O  # noqa: E402


def upd(u):
    if u.kind == 0:
        return P.RankOneUpdate.self_loop(u.i, u.rho)
    if u.kind == 1:
        return P.RankOneUpdate.edge_delta(u.i, u.j, u.rho)
    return P.RankOneUpdate.general(u.v, u.rho)


ref = O.Reference()
res = {"metric": "max over the batch of max_i |y_i - r_i| / max_i |r_i| per signal",
       "reference": "oracle/_ref (the reference's headers compiled in place, FFTW stand-in), all host threads",
       "ozaki_slices_n8192": P.ozaki_slices(8192), "cases": {}}
for cid in (1, 2, 3, 4, 5):
    cfg = O.config(cid)
    s = ref.fill(cfg.seed, cfg.dist, cfg.n, cfg.batch, cfg.r)
    t = time.time()
    if cfg.progressive:
        plan = P.PrunedEnsemblePlan(cfg.n, [upd(u) for u in cfg.updates], cfg.n, 1.7e308)
        want = ref.ensemble(cfg.n, list(cfg.updates), cfg.n, float(np.finfo(np.float64).max)).forward_all(s)
        for dt in ("float32", "float64"):
            got = plan.forward_all_batch(torch.as_tensor(s, device="cuda").to(getattr(torch, dt))).double().cpu().numpy()
            res["cases"][f"C{cid} forward_all {dt} ({cfg.batch} x 17 sets)"] = max(
                O.parity(got[:, r, :], want[:, r, :]) for r in range(17))
        continue
    plan = P.DctPlusPlan(cfg.n, upd(cfg.updates[0]), 1e-12)
    rp = ref.plan(cfg.n, cfg.updates[0])
    want = rp.forward(s)
    for dt in ("float64", "float32"):
        if cid == 5 and dt == "float32":
            continue
        got = plan.forward(torch.as_tensor(s, device="cuda").to(getattr(torch, dt))).double().cpu().numpy()
        res["cases"][f"C{cid} forward {dt} ({cfg.batch})"] = O.parity(got, want)
    if cid in (3, 5):
        back = rp.inverse(want)
        for dt in ("float64", "float32"):
            if cid == 5 and dt == "float32":
                continue
            got = plan.inverse(torch.as_tensor(want, device="cuda").to(getattr(torch, dt))).double().cpu().numpy()
            res["cases"][f"C{cid} inverse {dt} ({cfg.batch})"] = O.parity(got, back)
    mine, theirs = plan.setup(), rp.setup()
    res["cases"][f"C{cid} setup mu/sigma/slots bit-equal"] = bool(
        np.array_equal(mine["mu"], theirs["mu"]) and np.array_equal(mine["sigma"], theirs["sigma"]) and
        np.array_equal(mine["slot_pass"], theirs["slot_pass"]))
    print(cid, round(time.time() - t, 1), flush=True)
json.dump(res, open(sys.argv[1], "w"), indent=1)
print(json.dumps(res, indent=1))
