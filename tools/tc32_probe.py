#!/usr/bin/env python3
"""tcgen05 3xTF32 progressive GEMM (C4) against the FFMA SGEMM route and
the reference's forward_all on a slice: max-norm relative error and timing.
python tools/tc32_probe.py [batch]"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2409_08970_b200 as P  # noqa: E402
from oracle import checkers as O  # noqa: E402


def run(plan, x, out, mode):
    os.environ["DCTP_TC32"] = mode
    P.profile_reset()
    P.profile_enable(True)
    plan.forward_all_batch(x, out=out)
    P.profile_enable(False)
    kern = sorted(P.profile_summary())
    for _ in range(3):
        plan.forward_all_batch(x, sync=False, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        plan.forward_all_batch(x, sync=False, out=out)
    e1.record()
    torch.cuda.synchronize()
    return kern, e0.elapsed_time(e1) / 10


def main():
    batch = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    cfg = O.config(4)
    ups = [P.RankOneUpdate.self_loop(u.i, u.rho) for u in cfg.updates]
    plan = P.PrunedEnsemblePlan(cfg.n, ups, cfg.n, 1e300)
    s = P.fill_signals(cfg.seed, cfg.dist, cfg.n, batch, cfg.r)
    x = torch.as_tensor(s, device="cuda").float()
    outs = {}
    for mode in ("0", "1"):
        out = torch.empty((batch, 17, cfg.n), dtype=torch.float32, device="cuda")
        kern, ms = run(plan, x, out, mode)
        outs[mode] = out.double().cpu().numpy()
        print(f"DCTP_TC32={mode}: {kern} {ms:.4f} ms, {batch * 16 * cfg.n / ms * 1e3:.3e} samples/s", flush=True)
    a, b = outs["1"], outs["0"]
    print("tc32 vs sgemm max-norm rel:", float((np.abs(a - b).max(axis=(1, 2)) / np.abs(b).max(axis=(1, 2))).max()))
    try:
        ref = O.Reference().ensemble(cfg.n, [O.Update(u.kind, u.rho, u.i, u.j) for u in cfg.updates], cfg.n,
                                     float(np.finfo(np.float64).max))
        want = ref.forward_all(s[:512])
        for mode, o in outs.items():
            print(f"DCTP_TC32={mode} vs reference (512 rows):", O.parity(o[:512].reshape(512, -1), want.reshape(512, -1)))
    except Exception as e:  # noqa: BLE001
        print("reference:", e)


if __name__ == "__main__":
    main()
