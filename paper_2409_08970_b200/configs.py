"""The five BASELINE.json workloads, as reference API calls (SURVEY.md 8,
"Config -> reference API mapping").  BASELINE vertices are 0-based; the
reference's RankOneUpdate is 1-based.  Seeds: mix_seed(2409, n, config_id)
(SURVEY.md 8c); signals are drawn with the reference's Rng (signal.hpp)."""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache
from typing import Tuple

import numpy as np

SEED = 2409


@dataclass(frozen=True)
class Workload:
    cid: int
    name: str
    n: int
    batch: int
    dist: int          # fill_signals distribution id
    r: float           # AR coefficient where the distribution has one
    updates: Tuple     # ((kind, rho, i, j), ...) 1-based; kind 2 = general (direction below)
    dtypes: Tuple[str, ...]
    inverse: bool = False
    chain: bool = False  # rank-k chain (compose_rank_k) instead of an ensemble

    @property
    def progressive(self) -> bool:
        return len(self.updates) > 1 and not self.chain

    @property
    def seed(self) -> int:
        from .dctplus import mix_seed

        return mix_seed(SEED, self.n, self.cid)


@lru_cache(maxsize=None)
def general_direction(n: int = 8192) -> np.ndarray:
    """Config 5: u_i = gaussian() / sqrt(n) from Rng(mix_seed(2409, n, 50))."""
    from .dctplus import fill_signals, mix_seed

    return fill_signals(mix_seed(SEED, n, 50), 0, n, 1)[0] / np.sqrt(n)


WORKLOADS = {
    1: Workload(1, "C1 n=64 self_loop(1,0.5) fwd fp64 batch 4096", 64, 4096, 0, 0.0, ((0, 0.5, 1, 0),), ("f64",)),
    2: Workload(2, "C2 n=256 edge_delta(128,129,-0.7) fwd fp64 batch 65536", 256, 65536, 2, 0.95,
                ((1, -0.7, 128, 129),), ("f64",)),
    3: Workload(3, "C3 n=1024 edge_delta(1,1024,1.0) fwd+inv fp64/fp32 batch 16384", 1024, 16384, 3, 0.0,
                ((1, 1.0, 1, 1024),), ("f64", "f32"), inverse=True),
    4: Workload(4, "C4 n=128 K=16 self_loop(1,w_k) progressive fp32 batch 65536", 128, 65536, 4, 0.9,
                tuple((0, 0.05 + k * (1.95 / 15.0), 1, 0) for k in range(16)), ("f32",)),
    5: Workload(5, "C5 n=8192 general u~N(0,1/n) rho=0.1 fwd fp64 batch 2048", 8192, 2048, 0, 0.0,
                ((2, 0.1, 0, 0),), ("f64",)),
    # not a BASELINE config: the rank-k chain row of SURVEY.md 8(f)
    6: Workload(6, "X6 n=1024 chain self_loop(1,1.5)+edge_delta(1,1024,-0.5)+edge_delta(300,700,0.25) fwd fp64 "
                   "batch 16384", 1024, 16384, 2, 0.95,
                ((0, 1.5, 1, 0), (1, -0.5, 1, 1024), (1, 0.25, 300, 700)), ("f64",), chain=True),
    # not BASELINE configs: the NFST fast route where the
    # reference's own forward() is its NFST approximation — 7: it lies 5e-9 from
    # the exact transform (the plan keeps the NFST route for fidelity); 8: the
    # NFST route is also the faster one (n = 2048, fully kept)
    7: Workload(7, "X7 n=1024 self_loop(1,0.5) fwd fp64 batch 16384 (NFST route)", 1024, 16384, 0, 0.0,
                ((0, 0.5, 1, 0),), ("f64",)),
    8: Workload(8, "X8 n=2048 self_loop(1,5.0) fwd fp64 batch 8192 (NFST route)", 2048, 8192, 0, 0.0,
                ((0, 5.0, 1, 0),), ("f64",)),
}


def make_update(u):
    from .dctplus import RankOneUpdate

    kind, rho, i, j = u
    if kind == 0:
        return RankOneUpdate.self_loop(i, rho)
    if kind == 1:
        return RankOneUpdate.edge_delta(i, j, rho)
    return RankOneUpdate.general(general_direction(), rho)


def make_plan(w: Workload, device: int = 0):
    from .dctplus import ChainedFactorization, DctPlusPlan, PrunedEnsemblePlan

    if w.chain:
        return ChainedFactorization(w.n, [make_update(u) for u in w.updates], device=device)
    if w.progressive:
        return PrunedEnsemblePlan(w.n, [make_update(u) for u in w.updates], w.n, 1.7e308, device=device)
    return DctPlusPlan(w.n, make_update(w.updates[0]), 1e-12, device=device)
