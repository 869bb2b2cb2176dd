#!/usr/bin/env python3
"""Per-graph setup time (plan creation) with the secular roots / normalisers
on the host (DCTP_GPU_SETUP=0) or the GPU (=1): C5 (n = 8192 general
direction) and C3 (n = 1024).  python tools/setup_time.py"""
import json
import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2409_08970_b200 as P  # noqa: E402
from oracle import checkers as O  # noqa: E402


def main():
    torch.cuda.init()
    P.DctPlusPlan(64, P.RankOneUpdate.self_loop(1, 0.5), 1e-12)  # context, pool
    for cid in (3, 5):
        cfg = O.config(cid)
        u = cfg.updates[0]
        pu = (P.RankOneUpdate.general(u.v, u.rho) if u.kind == 2 else P.RankOneUpdate.edge_delta(u.i, u.j, u.rho))
        res = {"config": cid, "n": cfg.n, "threads": os.cpu_count()}
        for mode in ("0", "1"):
            os.environ["DCTP_GPU_SETUP"] = mode
            t = time.perf_counter()
            P.DctPlusPlan(cfg.n, pu, 1e-12)
            torch.cuda.synchronize()
            res["gpu" if mode == "1" else "host"] = round(time.perf_counter() - t, 4)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
