"""Per-config kernel timing (device-resident inputs, CUDA events), one JSON
line per config/direction/dtype.  Development tool; bench.py is the contract."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2409_08970_b200 as P  # noqa: E402
from oracle import checkers as O  # noqa: E402


def upd(u):
    if u.kind == 0:
        return P.RankOneUpdate.self_loop(u.i, u.rho)
    if u.kind == 1:
        return P.RankOneUpdate.edge_delta(u.i, u.j, u.rho)
    return P.RankOneUpdate.general(u.v, u.rho)


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def main(cids):
    for cid in cids:
        cfg = O.config(cid)
        t0 = time.time()
        if cfg.progressive:
            plan = P.PrunedEnsemblePlan(cfg.n, [upd(u) for u in cfg.updates], cfg.n, 1e300)
        else:
            plan = P.DctPlusPlan(cfg.n, upd(cfg.updates[0]), 1e-12)
        setup_s = time.time() - t0
        s64 = torch.as_tensor(P.fill_signals(cfg.seed, cfg.dist, cfg.n, cfg.batch, cfg.r), device="cuda")
        for dt in cfg.dtypes:
            s = s64 if dt == "f64" else s64.float()
            if cfg.progressive:
                out = torch.empty((cfg.batch, 17, cfg.n), dtype=s.dtype, device="cuda")
                ms = timeit(lambda: plan.forward_all_batch(s, sync=False, out=out))
                samples = cfg.batch * 16 * cfg.n
                runs = [("forward_all", ms, samples)]
            else:
                out = torch.empty_like(s)
                ms = timeit(lambda: plan.forward(s, sync=False, out=out))
                runs = [("forward", ms, cfg.batch * cfg.n)]
                if cfg.inverse:
                    ms_i = timeit(lambda: plan.inverse(s, sync=False, out=out))
                    runs.append(("inverse", ms_i, cfg.batch * cfg.n))
            for name, ms, samples in runs:
                print(json.dumps({"config": cid, "op": name, "dtype": dt, "ms": round(ms, 4),
                                  "samples_per_s": samples / (ms * 1e-3), "setup_s": round(setup_s, 3)}), flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5])
