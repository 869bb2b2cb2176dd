"""ORACLE TEST INFRASTRUCTURE — writes tests/golden/*.npz from the reference.

Run here (where /root/reference exists):  python oracle/gen_golden.py
The fixtures are committed; the GPU box never needs /root/reference.

Per BASELINE config (oracle.configs()):
  setup vectors of every member plan: lambda, z (deflated), mu, a, sigma,
  slot_pass, slot_idx, sub_mu, slow_path           (fast_transform.hpp:45-134)
  the first `rows` signals of the seeded batch (regenerable from seed/dist)
  forward outputs of DctPlusPlan::forward           (:163-190)
  C3: inverse(forward(s)) and inverse of a seeded p (:218-255)
  C4: PrunedEnsemblePlan(128, ups, 128, DBL_MAX).forward_all (:396-439)
plus known-answer cases from the reference's tests (test_cauchy.cpp:91-100,
test_spectral.cpp:55-61, :129-135, test_trig.cpp:72-77, test_fast_transform.cpp:213-250).
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import checkers as O  # noqa: E402

OUT = ROOT / "tests" / "golden"
ROWS = {1: 64, 2: 32, 3: 16, 4: 16, 5: 4}
DBL_MAX = float(np.finfo(np.float64).max)


def setup_arrays(prefix: str, st: dict) -> dict:
    out = {}
    for k in ("lambda", "z", "mu", "a", "sigma", "slot_pass", "slot_idx", "sub_mu"):
        out[f"{prefix}{k}"] = st[k]
    out[f"{prefix}slow_path"] = np.array(st["slow_path"])
    return out


def gen_config(ref: O.Reference, rs: O.Restatement, cfg: O.Config) -> dict:
    rows = ROWS[cfg.cid]
    s = rs.signals(cfg, rows)
    data = {"n": np.array(cfg.n), "seed": np.array(cfg.seed, dtype=np.uint64), "dist": np.array(cfg.dist),
            "r": np.array(cfg.r), "signals": s}
    if cfg.progressive:
        ens = ref.ensemble(cfg.n, cfg.updates, cfg.n, DBL_MAX)
        data["forward_all"] = ens.forward_all(s)
        data["rhos"] = np.array([u.rho for u in cfg.updates])
        for r in range(1, len(cfg.updates) + 1):
            m = ens.member(r)
            data.update(setup_arrays(f"m{r}_", m.setup()))
            data[f"m{r}_forward"] = m.forward(s)
        return data
    u = cfg.updates[0]
    t = time.time()
    plan = ref.plan(cfg.n, u)
    print(f"  C{cfg.cid} reference setup {time.time() - t:.1f} s", flush=True)
    data.update(setup_arrays("", plan.setup()))
    if u.kind == 2:
        data["v"] = np.asarray(u.v)
    data["forward"] = plan.forward(s)
    if not data["slow_path"]:
        data["forward_nmvp"] = plan.forward(s, nmvp=True)
    if cfg.inverse:
        data["inverse_of_forward"] = plan.inverse(data["forward"])
        p = rs.fill_signals(O.mix_seed(O.SEED, cfg.n, 100 + cfg.cid), 0, cfg.n, rows)
        data["p"] = p
        data["inverse"] = plan.inverse(p)
    return data


def gen_kat(ref: O.Reference) -> dict:
    """Small reference cases (n = 2..33) used as known-answer / edge tests."""
    cases = {
        "selfloop_n2": (2, O.Update(0, 1.0, 1)),
        "selfloop_n3": (3, O.Update(0, 1.5, 2)),
        "edge_n4": (4, O.Update(1, 1.5, 2, 3)),
        "edge_n12_deflating": (12, O.Update(1, 1.5, 2, 3)),
        "neg_rho_n8": (8, O.Update(0, -0.7, 3)),
        "neg_rho_n33": (33, O.Update(1, -0.4, 5, 9)),
        "neg_rho_n64": (64, O.Update(0, -0.9, 1)),
        "edge_n16_far": (16, O.Update(1, 2.0, 1, 16)),
        "selfloop_n100": (100, O.Update(0, 3.0, 50)),
        "disconnect_n16": (16, O.Update(1, -1.0, 8, 9)),
    }
    out = {}
    rs = O.Restatement()
    for name, (n, u) in cases.items():
        plan = ref.plan(n, u)
        st = plan.setup()
        s = rs.fill_signals(O.mix_seed(O.SEED, n, 7), 2, n, 8, 0.99)
        out.update({f"{name}/{k}": v for k, v in setup_arrays("", st).items()})
        out[f"{name}/n"] = np.array(n)
        out[f"{name}/update"] = np.array([u.kind, u.rho, u.i, u.j], dtype=np.float64)
        out[f"{name}/signals"] = s
        out[f"{name}/forward"] = plan.forward(s)
        out[f"{name}/inverse_of_forward"] = plan.inverse(out[f"{name}/forward"])
    # trig KATs through the reference TrigPlan (trig.hpp:95-114)
    x = rs.fill_signals(O.mix_seed(O.SEED, 0, 8), 0, 64, 4)
    for n in (2, 4, 8, 12, 16, 17, 64):
        out[f"trig/dct2_{n}"] = ref.trig(0, x[:, :n])
        out[f"trig/idct2_{n}"] = ref.trig(1, x[:, :n])
        out[f"trig/in_{n}"] = x[:, :n].copy()
    return out


def main(only=None):
    OUT.mkdir(parents=True, exist_ok=True)
    ref, rs = O.Reference(), O.Restatement()
    for cfg in O.configs():
        if only and cfg.cid not in only:
            continue
        t = time.time()
        data = gen_config(ref, rs, cfg)
        np.savez_compressed(OUT / f"c{cfg.cid}.npz", **data)
        print(f"C{cfg.cid}: {time.time() - t:.1f} s", flush=True)
    if not only or 0 in only:
        np.savez_compressed(OUT / "kat.npz", **gen_kat(ref))
        print("kat done")


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or None)
