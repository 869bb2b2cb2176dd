"""ORACLE TEST INFRASTRUCTURE — Python access to the two CPU checkers.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
leg may import this module, and only as the checker (never as the product).

* ``Restatement`` — oracle/build/liboracle.so, the plain-C restatement of the
  reference's DCT+ path (oracle/dctp_oracle.c).  Always buildable (gcc).
* ``Reference``   — oracle/_ref/libdctref.so, the reference's own headers
  compiled in place with the FFTW stand-in (oracle/build_ref.sh).  Built here
  when /root/reference is present; the prebuilt file travels to the GPU box.

Configs of BASELINE.json (0-based vertices there, 1-based here):
  C1 n=64   self_loop(1, 0.5)                 N(0,1) rows, 4096 signals
  C2 n=256  edge_delta(128, 129, -0.7)        AR(1) 0.95 rows, 65536 signals
  C3 n=1024 edge_delta(1, 1024, 1.0)          2u-1 rows, 16384 signals, fwd+inv
  C4 n=128  16 x self_loop(1, 0.05+k*1.95/15) 2-D AR(1) 0.9 rows, 65536 signals
  C5 n=8192 general u_i = N(0,1)/sqrt(n), rho = 0.1, N(0,1) rows, 2048 signals
"""
from __future__ import annotations

import ctypes as C
import subprocess
from dataclasses import dataclass
from pathlib import Path
from typing import List, Optional, Sequence

import numpy as np

HERE = Path(__file__).resolve().parent
RESTATEMENT_LIB = HERE / "build" / "liboracle.so"
REFERENCE_LIB = HERE / "_ref" / "libdctref.so"

SEED = 2409  # mix_seed(2409, n, config_id)


def build(quiet: bool = True) -> None:
    """make -C oracle (restatement always; the reference when present)."""
    subprocess.run(["make", "-C", str(HERE)], check=True,
                   stdout=subprocess.DEVNULL if quiet else None, stderr=subprocess.STDOUT if quiet else None)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------------- configs

@dataclass(frozen=True)
class Update:
    kind: int  # 0 self_loop, 1 edge_delta, 2 general
    rho: float
    i: int = 0
    j: int = 0
    v: Optional[tuple] = None

    def vec(self, n: int) -> Optional[np.ndarray]:
        return None if self.v is None else np.asarray(self.v, dtype=np.float64)


@dataclass(frozen=True)
class Config:
    cid: int
    n: int
    batch: int
    dist: int  # fill_signals distribution id
    r: float
    updates: tuple
    dtypes: tuple
    inverse: bool = False

    @property
    def seed(self) -> int:
        return mix_seed(SEED, self.n, self.cid)

    @property
    def progressive(self) -> bool:
        return len(self.updates) > 1


def mix_seed(seed: int, size: int, kind: int) -> int:
    x = (seed * 0x9E3779B97F4A7C15 + size * 0x100000001B3 + kind + 1) & (2**64 - 1)
    x ^= x >> 33
    x = (x * 0xFF51AFD7ED558CCD) & (2**64 - 1)
    x ^= x >> 33
    return x


def c5_direction(n: int = 8192) -> tuple:
    """u_i = gaussian()/sqrt(n) from Rng(mix_seed(2409, n, 50))."""
    g = Restatement().fill_signals(mix_seed(SEED, n, 50), 0, n, 1)[0]
    return tuple(float(x) for x in g / np.sqrt(n))


def configs() -> List[Config]:
    ws = [0.05 + k * (1.95 / 15.0) for k in range(16)]
    return [
        Config(1, 64, 4096, 0, 0.0, (Update(0, 0.5, 1),), ("f64",)),
        Config(2, 256, 65536, 2, 0.95, (Update(1, -0.7, 128, 129),), ("f64",)),
        Config(3, 1024, 16384, 3, 0.0, (Update(1, 1.0, 1, 1024),), ("f64", "f32"), inverse=True),
        Config(4, 128, 65536, 4, 0.9, tuple(Update(0, w, 1) for w in ws), ("f32",)),
        Config(5, 8192, 2048, 0, 0.0, (Update(2, 0.1, 0, 0, c5_direction()),), ("f64",)),
    ]


def config(cid: int) -> Config:
    return configs()[cid - 1]


# ----------------------------------------------------------------- restatement

class Restatement:
    """ctypes view of oracle/build/liboracle.so (oracle/dctp_oracle.c)."""

    _lib = None

    def __init__(self):
        if Restatement._lib is None:
            if not RESTATEMENT_LIB.exists():
                build()
            lib = C.CDLL(str(RESTATEMENT_LIB))
            lib.orc_mix_seed.restype = C.c_uint64
            lib.orc_mix_seed.argtypes = [C.c_uint64, C.c_size_t, C.c_size_t]
            lib.orc_fill_signals.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_size_t, C.c_size_t, C.c_void_p]
            lib.orc_dct2.argtypes = [C.c_size_t, C.c_void_p, C.c_void_p, C.c_size_t]
            lib.orc_idct2.argtypes = [C.c_size_t, C.c_void_p, C.c_void_p, C.c_size_t]
            lib.orc_setup.argtypes = [C.c_size_t, C.c_void_p, C.c_double, C.c_double] + [C.c_void_p] * 10
            lib.orc_forward.argtypes = [C.c_size_t] + [C.c_void_p] * 9 + [C.c_size_t]
            lib.orc_inverse.argtypes = [C.c_size_t] + [C.c_void_p] * 9 + [C.c_size_t]
            Restatement._lib = lib
        self.lib = Restatement._lib

    def mix_seed(self, seed, size, kind) -> int:
        return int(self.lib.orc_mix_seed(seed, size, kind))

    def fill_signals(self, seed: int, dist: int, n: int, rows: int, r: float = 0.0) -> np.ndarray:
        out = np.empty((rows, n))
        if self.lib.orc_fill_signals(seed, dist, r, n, rows, _ptr(out)) != 0:
            raise ValueError("unknown distribution")
        return out

    def dct2(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
        y = np.empty_like(x)
        self.lib.orc_dct2(x.shape[1], _ptr(x), _ptr(y), x.shape[0])
        return y

    def idct2(self, y: np.ndarray) -> np.ndarray:
        y = np.ascontiguousarray(np.atleast_2d(y), dtype=np.float64)
        x = np.empty_like(y)
        self.lib.orc_idct2(y.shape[1], _ptr(y), _ptr(x), y.shape[0])
        return x

    def setup(self, n: int, v: np.ndarray, rho: float, tau: float = 1e-12) -> dict:
        v = np.ascontiguousarray(v, dtype=np.float64)
        d = {k: np.empty(n) for k in ("lambda", "z", "mu", "a", "sigma", "sub_mu")}
        d["slot_pass"] = np.empty(n, dtype=np.int32)
        d["slot_idx"] = np.empty(n, dtype=np.int64)
        nsub = C.c_size_t()
        slow = C.c_int()
        rc = self.lib.orc_setup(n, _ptr(v), rho, tau, _ptr(d["lambda"]), _ptr(d["z"]), _ptr(d["mu"]), _ptr(d["a"]),
                                _ptr(d["sigma"]), _ptr(d["slot_pass"]), _ptr(d["slot_idx"]), _ptr(d["sub_mu"]),
                                C.byref(nsub), C.byref(slow))
        if rc != 0:
            raise RuntimeError(f"orc_setup failed with status {rc}")
        d["sub_mu"] = d["sub_mu"][: nsub.value].copy()
        d["slow_path"] = bool(slow.value)
        return d

    def _apply(self, fn, st: dict, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
        n = x.shape[1]
        sub_mu = np.ascontiguousarray(st["sub_mu"]) if len(st["sub_mu"]) else np.zeros(1)
        out = np.empty_like(x)
        fn(n, _ptr(np.ascontiguousarray(st["lambda"])), _ptr(np.ascontiguousarray(st["z"])),
           _ptr(np.ascontiguousarray(st["a"])), _ptr(np.ascontiguousarray(st["sigma"])),
           _ptr(np.ascontiguousarray(st["slot_pass"], dtype=np.int32)),
           _ptr(np.ascontiguousarray(st["slot_idx"], dtype=np.int64)), _ptr(sub_mu), _ptr(x), _ptr(out), x.shape[0])
        return out

    def forward(self, st: dict, s: np.ndarray) -> np.ndarray:
        return self._apply(self.lib.orc_forward, st, s)

    def inverse(self, st: dict, p: np.ndarray) -> np.ndarray:
        return self._apply(self.lib.orc_inverse, st, p)

    def signals(self, cfg: Config, rows: int) -> np.ndarray:
        return self.fill_signals(cfg.seed, cfg.dist, cfg.n, rows, cfg.r)


def direction(u: Update, n: int) -> np.ndarray:
    if u.kind == 2:
        return np.asarray(u.v, dtype=np.float64)
    v = np.zeros(n)
    v[u.i - 1] = 1.0
    if u.kind == 1:
        v[u.j - 1] = -1.0
    return v


# ------------------------------------------------------------------- reference

class ReferenceUnavailable(RuntimeError):
    pass


class Reference:
    """ctypes view of oracle/_ref/libdctref.so (the reference headers, compiled)."""

    _lib = None

    def __init__(self):
        if Reference._lib is None:
            if not REFERENCE_LIB.exists():
                build()
            if not REFERENCE_LIB.exists():
                raise ReferenceUnavailable(f"{REFERENCE_LIB} not built (reference absent)")
            lib = C.CDLL(str(REFERENCE_LIB))
            lib.ref_last_error.restype = C.c_char_p
            lib.ref_plan_create.argtypes = [C.c_size_t, C.c_int, C.c_size_t, C.c_size_t, C.c_double, C.c_void_p,
                                            C.c_double, C.c_double, C.POINTER(C.c_void_p)]
            lib.ref_plan_destroy.argtypes = [C.c_void_p]
            lib.ref_plan_slow_path.argtypes = [C.c_void_p]
            lib.ref_plan_setup.argtypes = [C.c_void_p] + [C.c_void_p] * 9
            lib.ref_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int]
            lib.ref_inverse.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int]
            lib.ref_ensemble_create.argtypes = [C.c_size_t, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p,
                                                C.c_void_p, C.c_void_p, C.c_size_t, C.c_double, C.c_double,
                                                C.POINTER(C.c_void_p)]
            lib.ref_ensemble_destroy.argtypes = [C.c_void_p]
            lib.ref_ensemble_member.restype = C.c_void_p
            lib.ref_ensemble_member.argtypes = [C.c_void_p, C.c_size_t]
            lib.ref_ensemble_forward_all.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                                     C.c_int]
            lib.ref_ensemble_forward_all_bounds.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                            C.c_void_p, C.c_size_t, C.c_int]
            lib.ref_rdo_select.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]
            lib.ref_calibrate_prune_threshold.restype = C.c_double
            lib.ref_calibrate_prune_threshold.argtypes = [C.c_size_t, C.c_double, C.c_double, C.c_size_t,
                                                          C.c_uint64]
            lib.ref_chain_create.argtypes = [C.c_size_t, C.c_size_t] + [C.c_void_p] * 7 + [C.c_double,
                                                                                         C.POINTER(C.c_void_p)]
            lib.ref_chain_destroy.argtypes = [C.c_void_p]
            lib.ref_chain_spectrum.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_size_t)]
            lib.ref_chain_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
            lib.ref_format_update.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
            lib.ref_csv_row.argtypes = [C.c_char_p, C.c_size_t, C.c_char_p, C.c_char_p, C.c_char_p, C.c_double,
                                        C.c_char_p, C.c_size_t]
            lib.ref_trig.argtypes = [C.c_int, C.c_size_t, C.c_void_p, C.c_void_p, C.c_size_t]
            lib.ref_mix_seed.restype = C.c_uint64
            lib.ref_mix_seed.argtypes = [C.c_uint64, C.c_size_t, C.c_size_t]
            lib.ref_rng_fill.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_size_t, C.c_size_t, C.c_void_p]
            Reference._lib = lib
        self.lib = Reference._lib

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.lib.ref_last_error().decode()}")

    def plan(self, n: int, u: Update, eps: float = 1e-12, tau: float = 1e-12) -> "RefPlan":
        v = u.vec(n)
        h = C.c_void_p()
        self._check(self.lib.ref_plan_create(n, u.kind, u.i, u.j, u.rho, _ptr(v), eps, tau, C.byref(h)))
        return RefPlan(self, h, n, owned=True)

    def ensemble(self, n: int, ups: Sequence[Update], cp: int, thr: float, eps: float = 1e-12) -> "RefEnsemble":
        k = len(ups)
        kinds = np.array([u.kind for u in ups], dtype=np.int32)
        is_ = np.array([u.i for u in ups], dtype=np.uint64)
        js = np.array([u.j for u in ups], dtype=np.uint64)
        rhos = np.array([u.rho for u in ups], dtype=np.float64)
        vs = None
        if any(u.kind == 2 for u in ups):
            vs = np.stack([direction(u, n) for u in ups])
        h = C.c_void_p()
        self._check(self.lib.ref_ensemble_create(n, k, _ptr(kinds), _ptr(is_), _ptr(js), _ptr(rhos), _ptr(vs), cp,
                                                 thr, eps, C.byref(h)))
        return RefEnsemble(self, h, n, k)

    def chain(self, n: int, ups: Sequence[Update], base=None, tau: float = 1e-12) -> "RefChain":
        """compose_rank_k(base or path_spectrum(n), ups, tau); base = (lambda, u)."""
        kinds = np.array([u.kind for u in ups], dtype=np.int32)
        is_ = np.array([u.i for u in ups], dtype=np.uint64)
        js = np.array([u.j for u in ups], dtype=np.uint64)
        rhos = np.array([u.rho for u in ups], dtype=np.float64)
        vs = np.stack([direction(u, n) for u in ups]) if any(u.kind == 2 for u in ups) else None
        bl = bu = None
        if base is not None:
            bl = np.ascontiguousarray(base[0], dtype=np.float64)
            bu = np.ascontiguousarray(base[1], dtype=np.float64)
        h = C.c_void_p()
        self._check(self.lib.ref_chain_create(n, len(ups), _ptr(kinds), _ptr(is_), _ptr(js), _ptr(rhos), _ptr(vs),
                                              _ptr(bl), _ptr(bu), tau, C.byref(h)))
        return RefChain(self, h, n)

    def trig(self, kind: int, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
        y = np.empty_like(x)
        self._check(self.lib.ref_trig(kind, x.shape[1], _ptr(x), _ptr(y), x.shape[0]))
        return y

    def fill(self, seed: int, dist: int, n: int, rows: int, r: float = 0.0) -> np.ndarray:
        out = np.empty((rows, n))
        self.lib.ref_rng_fill(seed, dist, r, n, rows, _ptr(out))
        return out


class RefPlan:
    def __init__(self, ref: Reference, h, n: int, owned: bool):
        self.ref, self.h, self.n, self.owned = ref, h, n, owned

    def __del__(self):
        if self.owned and self.h is not None:
            self.ref.lib.ref_plan_destroy(self.h)
            self.h = None

    def slow_path(self) -> bool:
        return bool(self.ref.lib.ref_plan_slow_path(self.h))

    def setup(self) -> dict:
        n = self.n
        d = {k: np.empty(n) for k in ("lambda", "z", "mu", "a", "sigma", "sub_mu")}
        d["slot_pass"] = np.empty(n, dtype=np.int32)
        d["slot_idx"] = np.empty(n, dtype=np.int64)
        nsub = C.c_size_t()
        self.ref.lib.ref_plan_setup(self.h, _ptr(d["lambda"]), _ptr(d["z"]), _ptr(d["mu"]), _ptr(d["a"]),
                                    _ptr(d["sigma"]), _ptr(d["slot_pass"]), _ptr(d["slot_idx"]), _ptr(d["sub_mu"]),
                                    C.byref(nsub))
        d["sub_mu"] = d["sub_mu"][: nsub.value].copy()
        d["slow_path"] = self.slow_path()
        return d

    def forward(self, s: np.ndarray, nmvp: bool = False, threads: int = 0) -> np.ndarray:
        s = np.ascontiguousarray(np.atleast_2d(s), dtype=np.float64)
        out = np.empty_like(s)
        self.ref._check(self.ref.lib.ref_forward(self.h, _ptr(s), _ptr(out), s.shape[0], 1 if nmvp else 0, threads))
        return out

    def inverse(self, p: np.ndarray, fast: bool = True, threads: int = 0) -> np.ndarray:
        p = np.ascontiguousarray(np.atleast_2d(p), dtype=np.float64)
        out = np.empty_like(p)
        self.ref._check(self.ref.lib.ref_inverse(self.h, _ptr(p), _ptr(out), p.shape[0], 1 if fast else 0, threads))
        return out


class RefEnsemble:
    def __init__(self, ref: Reference, h, n: int, k: int):
        self.ref, self.h, self.n, self.k = ref, h, n, k

    def __del__(self):
        if self.h is not None:
            self.ref.lib.ref_ensemble_destroy(self.h)
            self.h = None

    def member(self, r: int) -> RefPlan:
        return RefPlan(self.ref, C.c_void_p(self.ref.lib.ref_ensemble_member(self.h, r)), self.n, owned=False)

    def forward_all(self, s: np.ndarray, threads: int = 0) -> np.ndarray:
        s = np.ascontiguousarray(np.atleast_2d(s), dtype=np.float64)
        out = np.empty((s.shape[0], self.k + 1, self.n))
        self.ref._check(self.ref.lib.ref_ensemble_forward_all(self.h, _ptr(s), _ptr(out), None, s.shape[0], threads))
        return out

    def forward_all_bounds(self, s: np.ndarray, threads: int = 0):
        """Result of PrunedEnsemblePlan::forward_all per signal: coeffs
        (batch, K+1, n), bounds (batch, K+1), pruned flags (batch,)."""
        s = np.ascontiguousarray(np.atleast_2d(s), dtype=np.float64)
        out = np.empty((s.shape[0], self.k + 1, self.n))
        bounds = np.empty((s.shape[0], self.k + 1))
        pruned = np.empty(s.shape[0], dtype=np.int32)
        self.ref._check(self.ref.lib.ref_ensemble_forward_all_bounds(self.h, _ptr(s), _ptr(out), _ptr(bounds),
                                                                     _ptr(pruned), s.shape[0], threads))
        return out, bounds, pruned

    def rdo_select(self, s: np.ndarray):
        """rdo_select (l1) per signal: (index, pruned) int32 arrays."""
        s = np.ascontiguousarray(np.atleast_2d(s), dtype=np.float64)
        idx = np.empty(s.shape[0], dtype=np.int32)
        pr = np.empty(s.shape[0], dtype=np.int32)
        self.ref._check(self.ref.lib.ref_rdo_select(self.h, _ptr(s), _ptr(idx), _ptr(pr), s.shape[0]))
        return idx, pr


class RefChain:
    def __init__(self, ref: Reference, h, n: int):
        self.ref, self.h, self.n = ref, h, n

    def __del__(self):
        if self.h is not None:
            self.ref.lib.ref_chain_destroy(self.h)
            self.h = None

    def spectrum(self):
        """(mu, x, number of stages) of the ChainedFactorization."""
        mu, x, k = np.empty(self.n), np.empty((self.n, self.n)), C.c_size_t()
        self.ref.lib.ref_chain_spectrum(self.h, _ptr(mu), _ptr(x), C.byref(k))
        return mu, x, k.value

    def forward(self, s: np.ndarray, threads: int = 0) -> np.ndarray:
        s = np.ascontiguousarray(np.atleast_2d(s), dtype=np.float64)
        out = np.empty_like(s)
        self.ref._check(self.ref.lib.ref_chain_forward(self.h, _ptr(s), _ptr(out), s.shape[0], threads))
        return out


def parity(y: np.ndarray, ref: np.ndarray) -> float:
    """SURVEY.md 8d / BASELINE.md section 3: max over signals of
    max_i |y_i - r_i| / max_i |r_i| (norm-wise, per signal)."""
    y = np.asarray(y, dtype=np.float64).reshape(ref.shape[0], -1)
    r = np.asarray(ref, dtype=np.float64).reshape(ref.shape[0], -1)
    den = np.maximum(np.abs(r).max(axis=1), np.finfo(np.float64).tiny)
    return float((np.abs(y - r).max(axis=1) / den).max())
