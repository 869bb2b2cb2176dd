"""Loader for the committed golden fixtures (tests/golden/*.npz, written by
oracle/gen_golden.py from the reference compiled in place)."""
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def setup_of(g: dict, prefix: str = "") -> dict:
    keys = ("lambda", "z", "mu", "a", "sigma", "slot_pass", "slot_idx", "sub_mu", "slow_path")
    return {k: g[prefix + k] for k in keys}


def kat_cases() -> list:
    g = load_golden("kat")
    names = sorted({k.split("/")[0] for k in g if "/" in k and not k.startswith("trig/")})
    out = []
    for name in names:
        d = {k.split("/", 1)[1]: v for k, v in g.items() if k.startswith(name + "/")}
        d["name"] = name
        out.append(d)
    return out
