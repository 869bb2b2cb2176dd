#!/usr/bin/env python3
"""NFST route probe: parity of the GPU fast route against the reference's
forward() (and the reference's own distance from its dense route), plus a
device timing.  python tools/nfst_probe.py N KIND RHO [I J] [--rows R]"""
import argparse
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2409_08970_b200 as P  # noqa: E402
from oracle import checkers as O  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("n", type=int)
    ap.add_argument("kind", type=int)
    ap.add_argument("rho", type=float)
    ap.add_argument("i", type=int, nargs="?", default=1)
    ap.add_argument("j", type=int, nargs="?", default=0)
    ap.add_argument("--rows", type=int, default=96)
    ap.add_argument("--batch", type=int, default=0)
    a = ap.parse_args()
    os.environ.setdefault("DCTP_FAST", "1")
    u = O.Update(a.kind, a.rho, a.i, a.j)
    pu = P.RankOneUpdate.self_loop(a.i, a.rho) if a.kind == 0 else P.RankOneUpdate.edge_delta(a.i, a.j, a.rho)
    plan = P.DctPlusPlan(a.n, pu, 1e-12)
    s = np.random.default_rng(a.n + 7).standard_normal((a.rows, a.n))
    got = plan.forward(torch.as_tensor(s, device="cuda")).cpu().numpy()
    try:
        rp = O.Reference().plan(a.n, u)
        want, exact = rp.forward(s), rp.forward(s, nmvp=True)
        e = np.abs(got - want).max(1) / np.abs(want).max(1)
        print(f"vs reference forward: max {e.max():.3e} median {np.median(e):.3e}; "
              f"reference fast vs dense {O.parity(want, exact):.3e}; ours vs dense {O.parity(got, exact):.3e}")
    except O.ReferenceUnavailable as ex:
        print("reference unavailable:", ex)
    batch = a.batch or (1 << 24) // a.n
    x = torch.randn(batch, a.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        plan.forward(x, out=y, sync=False)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(10):
        plan.forward(x, out=y, sync=False)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 10
    print(f"n={a.n} batch={batch}: {ms:.4f} ms/launch, {batch * a.n / ms * 1e3:.3e} samples/s")


if __name__ == "__main__":
    main()
