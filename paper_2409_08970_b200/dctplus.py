"""Python mirror of the reference's transform API (proj/include/dctplus/).

Same names, argument meaning and error behaviour as the C++ reference:

=====================================  ==============================================
reference (C++)                        here
=====================================  ==============================================
RankOneUpdate::self_loop / edge_delta  RankOneUpdate.self_loop / .edge_delta (graph.hpp:94-104)
(extension, config 5)                  RankOneUpdate.general(v, rho)
DctPlusPlan(n, u, eps, tau)            DctPlusPlan(n, u, eps, tau, device=0) (fast_transform.hpp:45)
plan.forward(s) / forward_nmvp(s)      plan.forward(s) / plan.forward_nmvp(s)   (:163, :199)
plan.inverse(p, fast)                  plan.inverse(p, fast=True)               (:218)
size/epsilon/lambda/mu/slow_path/basis size()/epsilon()/lambda_()/mu()/slow_path()/basis()
PrunedEnsemblePlan(n, us, cp, thr, e)  PrunedEnsemblePlan(n, us, cp, thr, e)   (:343), c_p = n
forward_all(s) -> Result               forward_all(s) -> Result                 (:396-446)
plan_dctplus / forward / inverse       plan_dctplus / forward / inverse         (:304-319)
std::invalid_argument / domain_error   InvalidArgument(ValueError) / DomainError
=====================================  ==============================================

A signal is a 1-D sequence of n samples (the reference's std::vector) or,
batched, a 2-D array of rows.  Host inputs (lists, numpy arrays) return numpy
arrays and go through the synchronous host-buffer C entry points; CUDA torch
tensors stay on the device and run on the current torch stream (float64 or
float32).  Every call lands in the sm_100a kernels; nothing here computes a
transform itself.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from ._native import check, lib

try:  # torch is the device-memory / stream plumbing, never the compute path
    import torch
except ImportError:  # pragma: no cover - the image always has torch
    torch = None

SELF_LOOP, EDGE_DELTA, GENERAL = 0, 1, 2


@dataclass(frozen=True)
class RankOneUpdate:
    """L + rho v v^T on the path graph; vertices are 1-based (graph.hpp:87-114)."""

    kind: int
    rho: float
    node_i: int = 0
    node_j: int = 0
    v: Optional[tuple] = None

    @staticmethod
    def self_loop(i: int, w: float) -> "RankOneUpdate":
        if i < 1:
            raise N.InvalidArgument("RankOneUpdate: node index is 1-based")
        if w == 0.0:
            raise N.InvalidArgument("RankOneUpdate: weight must be nonzero")
        return RankOneUpdate(SELF_LOOP, float(w), int(i), 0)

    @staticmethod
    def edge_delta(i: int, j: int, w: float) -> "RankOneUpdate":
        if i < 1 or i >= j:
            raise N.InvalidArgument("RankOneUpdate: need 1 <= i < j")
        if w == 0.0:
            raise N.InvalidArgument("RankOneUpdate: weight must be nonzero")
        return RankOneUpdate(EDGE_DELTA, float(w), int(i), int(j))

    @staticmethod
    def general(v: Sequence[float], rho: float) -> "RankOneUpdate":
        """Extension beyond the reference: arbitrary direction v (config 5)."""
        if rho == 0.0:
            raise N.InvalidArgument("RankOneUpdate: weight must be nonzero")
        vv = tuple(float(x) for x in np.asarray(v, dtype=np.float64).ravel())
        if not vv:
            raise N.InvalidArgument("RankOneUpdate: empty direction")
        return RankOneUpdate(GENERAL, float(rho), 0, 0, vv)

    def direction(self, n: int) -> np.ndarray:
        if self.kind == GENERAL:
            if len(self.v) != n:
                raise N.InvalidArgument("RankOneUpdate: direction length mismatch")
            return np.array(self.v)
        if self.node_i > n or (self.kind == EDGE_DELTA and self.node_j > n):
            raise N.InvalidArgument("RankOneUpdate: node index exceeds graph size")
        out = np.zeros(n)
        out[self.node_i - 1] = 1.0
        if self.kind == EDGE_DELTA:
            out[self.node_j - 1] = -1.0
        return out

    def _v_ptr(self):
        if self.kind != GENERAL:
            return None, None
        arr = np.ascontiguousarray(self.v, dtype=np.float64)
        return arr, arr.ctypes.data_as(C.c_void_p)


def _is_device_tensor(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def _stream_ptr(device: int):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _as_rows(x, n: int, what: str):
    """Host path: numpy view of shape (batch, n) plus whether input was 1-D."""
    arr = np.asarray(x)
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    single = arr.ndim == 1
    rows = arr.reshape(1, -1) if single else arr
    if rows.ndim != 2 or rows.shape[1] != n:
        raise N.InvalidArgument(f"{what}: signal size mismatch")
    return np.ascontiguousarray(rows), single


def _dev_rows(x, n: int, what: str):
    if x.dtype not in (torch.float32, torch.float64):
        raise N.InvalidArgument(f"{what}: device signals must be float32 or float64")
    single = x.dim() == 1
    rows = x.reshape(1, -1) if single else x
    if rows.dim() != 2 or rows.shape[1] != n:
        raise N.InvalidArgument(f"{what}: signal size mismatch")
    return rows.contiguous(), single


def _check_out(out, rows, shape, what: str):
    """A caller-supplied device output: same dtype and device as the rows,
    contiguous, exactly `shape`, and not overlapping the input."""
    if not _is_device_tensor(out):
        raise N.InvalidArgument(f"{what}: out must be a CUDA tensor")
    if out.dtype != rows.dtype or out.device != rows.device:
        raise N.InvalidArgument(f"{what}: out must match the input's dtype and device")
    if out.dim() == len(shape) - 1 and shape[0] == 1:  # one signal: out without the batch axis
        out = out.unsqueeze(0)
    if tuple(out.shape) != tuple(shape):
        raise N.InvalidArgument(f"{what}: out has shape {tuple(out.shape)}, expected {tuple(shape)}")
    if not out.is_contiguous():
        raise N.InvalidArgument(f"{what}: out must be contiguous")
    a0, a1 = rows.data_ptr(), rows.data_ptr() + rows.numel() * rows.element_size()
    b0, b1 = out.data_ptr(), out.data_ptr() + out.numel() * out.element_size()
    if out.numel() and rows.numel() and a0 < b1 and b0 < a1:
        raise N.InvalidArgument(f"{what}: out must not overlap the input")
    return out


class DctPlusPlan:
    """Fast DCT+ of one rank-one update of the path graph (fast_transform.hpp:43-302)."""

    def __init__(self, n: int, update: RankOneUpdate, epsilon: float, tau: float = 1e-12, device: int = 0,
                 _handle=None, _owner=None):
        self._update = update
        if _handle is not None:  # ensemble member view
            self._h = _handle
            self._owner = _owner
        else:
            self._owner = None
            if n < 2:
                raise N.InvalidArgument("DctPlusPlan: need n >= 2")
            if update.kind == GENERAL:
                update.direction(n)  # length check: the C ABI reads exactly n doubles
            varr, vptr = update._v_ptr()
            h = C.c_void_p()
            check(lib.dctp_plan_create(n, update.kind, update.node_i, update.node_j, update.rho, vptr,
                                       float(epsilon), float(tau), int(device), C.byref(h)))
            self._h = h
        n_ = C.c_size_t()
        eps = C.c_double()
        slow = C.c_int()
        kept = C.c_size_t()
        act = C.c_size_t()
        dev = C.c_int()
        check(lib.dctp_plan_info(self._h, C.byref(n_), C.byref(eps), C.byref(slow), C.byref(kept), C.byref(act),
                                 C.byref(dev)))
        self._n, self._eps, self._slow = n_.value, eps.value, bool(slow.value)
        self.n_kept, self.n_active, self.device = kept.value, act.value, dev.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and getattr(self, "_owner", None) is None and lib is not None:
            lib.dctp_plan_destroy(h)
            self._h = None

    # --- accessors (fast_transform.hpp:136-143) ---------------------------------
    def size(self) -> int:
        return self._n

    def epsilon(self) -> float:
        return self._eps

    def update(self) -> RankOneUpdate:
        return self._update

    def slow_path(self) -> bool:
        return self._slow

    def route(self) -> dict:
        """fp64 forward route: {"nfst": bool, "probe_gap": float} (dctp_plan_route)."""
        f = C.c_int()
        g = C.c_double()
        check(lib.dctp_plan_route(self._h, C.byref(f), C.byref(g)))
        return {"nfst": bool(f.value), "probe_gap": g.value}

    def _setup(self):
        n = self._n
        out = {k: np.empty(n) for k in ("lambda", "mu", "z", "a", "sigma")}
        ptr = {k: v.ctypes.data_as(C.c_void_p) for k, v in out.items()}
        check(lib.dctp_plan_setup(self._h, ptr["lambda"], ptr["mu"], ptr["z"], ptr["a"], ptr["sigma"]))
        return out

    def lambda_(self) -> np.ndarray:
        return self._setup()["lambda"]

    def mu(self) -> np.ndarray:
        return self._setup()["mu"]

    def setup(self) -> dict:
        """lambda, mu, deflated z, per-slot a and sigma, slot map (factorization())."""
        d = self._setup()
        n = self._n
        pas = np.empty(n, dtype=np.int32)
        idx = np.empty(n, dtype=np.int64)
        check(lib.dctp_plan_slots(self._h, pas.ctypes.data_as(C.c_void_p), idx.ctypes.data_as(C.c_void_p)))
        d["slot_pass"], d["slot_idx"] = pas, idx
        return d

    def basis(self) -> np.ndarray:
        x = np.empty((self._n, self._n))
        check(lib.dctp_plan_basis(self._h, x.ctypes.data_as(C.c_void_p)))
        return x

    # --- apply -------------------------------------------------------------------
    _DEV = {("fwd", True): "dctp_forward_f64", ("fwd", False): "dctp_forward_f32",
            ("inv", True): "dctp_inverse_f64", ("inv", False): "dctp_inverse_f32",
            ("fwd_nmvp", True): "dctp_forward_nmvp_f64", ("fwd_nmvp", False): "dctp_forward_nmvp_f32",
            ("inv_nmvp", True): "dctp_inverse_nmvp_f64", ("inv_nmvp", False): "dctp_inverse_nmvp_f32"}

    def _apply(self, x, op: str, sync: bool = True, out=None):
        n = self._n
        what = "DctPlusPlan"
        if _is_device_tensor(x):
            rows, single = _dev_rows(x, n, what)
            y = _check_out(out, rows, rows.shape, what) if out is not None else torch.empty_like(rows)
            fn = getattr(lib, self._DEV[(op, rows.dtype == torch.float64)])
            stream = _stream_ptr(rows.device)
            check(fn(self._h, C.c_void_p(rows.data_ptr()), C.c_void_p(y.data_ptr()), rows.shape[0], stream))
            if sync:
                check(lib.dctp_plan_sync_check(self._h, stream))
            return y.reshape(-1) if single else y
        rows, single = _as_rows(x, n, what)
        y = np.empty_like(rows)
        name = self._DEV[(op, rows.dtype == np.float64)]
        fn = getattr(lib, name[:-4] + "_host" + name[-4:])
        check(fn(self._h, rows.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), rows.shape[0]))
        return y.reshape(-1) if single else y

    def forward(self, s, sync: bool = True, out=None):
        """Coefficients in ascending-eigenvalue slot order (fast_transform.hpp:163-195)."""
        return self._apply(s, "fwd", sync=sync, out=out)

    def forward_nmvp(self, s, sync: bool = True, out=None):
        """The reference's dense X^T s (:199-214): one product with the
        materialised basis on the fp64 tensor cores (built on first use)."""
        return self._apply(s, "fwd_nmvp", sync=sync, out=out)

    def inverse(self, p, fast: bool = True, sync: bool = True, out=None):
        """X p (:218-260): fast = the transposed Cauchy + DCT-III route,
        fast = False the dense product with the materialised basis."""
        return self._apply(p, "inv" if fast else "inv_nmvp", sync=sync, out=out)

    def sync_check(self):
        check(lib.dctp_plan_sync_check(self._h, _stream_ptr(torch.cuda.current_device())))


def plan_dctplus(n: int, u: RankOneUpdate, epsilon: float, tau: float = 1e-12, device: int = 0) -> DctPlusPlan:
    return DctPlusPlan(n, u, epsilon, tau, device)


def forward(plan: DctPlusPlan, s):
    return plan.forward(s)


def forward_nmvp(plan: DctPlusPlan, s):
    return plan.forward_nmvp(s)


def inverse(plan: DctPlusPlan, p):
    return plan.inverse(p)


@dataclass
class Result:
    """PrunedEnsemblePlan::Result (fast_transform.hpp:383-387)."""

    pruned: bool = False
    coeffs: List[np.ndarray] = field(default_factory=list)
    bounds: List[float] = field(default_factory=list)


def path_quadratic_form(s) -> float:
    """sum (s_i - s_{i+1})^2 (fast_transform.hpp:24-31) — host helper for Result.pruned."""
    a = np.asarray(s, dtype=np.float64)
    d = a[:-1] - a[1:]
    return float(np.cumsum(d * d)[-1]) if d.size else 0.0  # sequential, as the reference


class PrunedEnsemblePlan:
    """Shared DCT + K Cauchy stages (fast_transform.hpp:338-454): progressive
    (c_p = n) and pruned (c_p < n: signals whose path quadratic form is at
    most `threshold` keep c_p coefficients per set, with error bounds)."""

    kDenseMemberCutoff = 128

    def __init__(self, n: int, updates: Sequence[RankOneUpdate], cp: int, threshold: float,
                 epsilon: float = 1e-12, device: int = 0):
        k = len(updates)
        kinds = (C.c_int * max(k, 1))(*[u.kind for u in updates])
        is_ = (C.c_size_t * max(k, 1))(*[u.node_i for u in updates])
        js = (C.c_size_t * max(k, 1))(*[u.node_j for u in updates])
        rhos = (C.c_double * max(k, 1))(*[u.rho for u in updates])
        vs = None
        if any(u.kind == GENERAL for u in updates):
            for u in updates:
                if u.kind == GENERAL:
                    u.direction(n)
            vs = np.zeros((k, n))
            for r, u in enumerate(updates):
                if u.kind == GENERAL:
                    vs[r] = u.direction(n)
        h = C.c_void_p()
        check(lib.dctp_ensemble_create(n, k, kinds, is_, js, rhos,
                                       None if vs is None else vs.ctypes.data_as(C.c_void_p), cp,
                                       float(threshold), float(epsilon), int(device), C.byref(h)))
        self._h = h
        self._n, self._cp, self._thr, self._updates = n, cp, float(threshold), list(updates)
        self.device = device
        self._members = []
        for r in range(1, k + 1):
            m = C.c_void_p()
            check(lib.dctp_ensemble_member(h, r, C.byref(m)))
            self._members.append(DctPlusPlan(n, updates[r - 1], epsilon, _handle=m, _owner=self))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and lib is not None:
            self._members = []
            lib.dctp_ensemble_destroy(h)
            self._h = None

    def size(self) -> int:
        return self._n

    def keep_count(self) -> int:
        return self._cp

    def threshold(self) -> float:
        return self._thr

    def ensemble_size(self) -> int:
        return len(self._members) + 1

    def member(self, r: int) -> DctPlusPlan:
        if r < 1 or r > len(self._members):
            raise N.LogicError("PrunedEnsemblePlan::member: index out of range")
        return self._members[r - 1]

    def forward_all_batch(self, s, sync: bool = True, out=None, with_bounds: bool = False):
        """Batched forward_all: rows -> (batch, K+1, n); set 0 is the shared DCT.
        with_bounds=True also returns the truncation-error bounds (batch, K+1)
        and the pruned-branch flags (batch,) of Result (device rows only)."""
        n, sets = self._n, self.ensemble_size()
        if _is_device_tensor(s):
            rows, single = _dev_rows(s, n, "pruned_forward_all")
            y = _check_out(out, rows, (rows.shape[0], sets, n), "pruned_forward_all") if out is not None else \
                torch.empty((rows.shape[0], sets, n), dtype=rows.dtype, device=rows.device)
            stream = _stream_ptr(rows.device)
            if with_bounds:
                bounds = torch.empty((rows.shape[0], sets), dtype=rows.dtype, device=rows.device)
                pruned = torch.empty((rows.shape[0],), dtype=torch.uint8, device=rows.device)
                fn = lib.dctp_ensemble_forward_all_pruned_f64 if rows.dtype == torch.float64 else \
                    lib.dctp_ensemble_forward_all_pruned_f32
                check(fn(self._h, C.c_void_p(rows.data_ptr()), C.c_void_p(y.data_ptr()),
                         C.c_void_p(bounds.data_ptr()), C.c_void_p(pruned.data_ptr()), rows.shape[0], stream))
            else:
                fn = lib.dctp_ensemble_forward_all_f64 if rows.dtype == torch.float64 else \
                    lib.dctp_ensemble_forward_all_f32
                check(fn(self._h, C.c_void_p(rows.data_ptr()), C.c_void_p(y.data_ptr()), rows.shape[0], stream))
            if sync:
                check(lib.dctp_ensemble_sync_check(self._h, stream))
            if with_bounds:
                return (y[0], bounds[0], pruned[0]) if single else (y, bounds, pruned)
            return y[0] if single else y
        if with_bounds:
            raise N.InvalidArgument("forward_all_batch(with_bounds=True) takes device rows; use forward_all")
        rows, single = _as_rows(s, n, "pruned_forward_all")
        y = np.empty((rows.shape[0], sets, n), dtype=rows.dtype)
        fn = lib.dctp_ensemble_forward_all_host_f64 if rows.dtype == np.float64 else \
            lib.dctp_ensemble_forward_all_host_f32
        check(fn(self._h, rows.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), rows.shape[0]))
        return y[0] if single else y

    def forward_all(self, s) -> Result:
        """One signal -> Result{pruned, coeffs[K+1], bounds} (fast_transform.hpp:396-446).
        With c_p = n both branches give the exact K+1 coefficient sets and
        zero truncation bounds."""
        a = np.ascontiguousarray(np.asarray(s, dtype=np.float64))
        if a.ndim != 1 or a.shape[0] != self._n:
            raise N.InvalidArgument("pruned_forward_all: size mismatch")
        sets = self.ensemble_size()
        coeffs = np.empty((sets, self._n))
        bounds = np.empty(sets)
        pruned = (C.c_ubyte * 1)()
        check(lib.dctp_ensemble_forward_all_pruned_host_f64(self._h, a.ctypes.data_as(C.c_void_p),
                                                            coeffs.ctypes.data_as(C.c_void_p),
                                                            bounds.ctypes.data_as(C.c_void_p), pruned, 1))
        return Result(pruned=bool(pruned[0]), coeffs=[c for c in coeffs], bounds=[float(b) for b in bounds])


def plan_pruned(n, updates, cp, threshold, epsilon=1e-12, device=0) -> PrunedEnsemblePlan:
    return PrunedEnsemblePlan(n, updates, cp, threshold, epsilon, device)


def pruned_forward_all(plan: PrunedEnsemblePlan, s) -> Result:
    return plan.forward_all(s)


@dataclass
class RdoChoice:
    """fast_transform.hpp:466-470."""

    index: int = 0
    coeffs: np.ndarray = None
    pruned: bool = False


def rdo_select(plan: PrunedEnsemblePlan, s, cost=None) -> RdoChoice:
    """The ensemble member whose coefficients minimise `cost` (default l1,
    the reference's rate-distortion proxy), ties to the lower index, on the
    pruned or full outputs per the threshold branch (fast_transform.hpp:472-496)."""
    res = plan.forward_all(s)
    cost = cost or (lambda c: float(np.abs(c).sum()))
    best, idx = cost(res.coeffs[0]), 0
    for r in range(1, len(res.coeffs)):
        c = cost(res.coeffs[r])
        if c < best:
            best, idx = c, r
    return RdoChoice(index=idx, coeffs=res.coeffs[idx], pruned=res.pruned)


def rdo_select_batch(plan: PrunedEnsemblePlan, rows, sync: bool = True):
    """rdo_select (l1 cost) for device rows on the GPU: (index int32 (batch,),
    chosen coefficients (batch, n), pruned uint8 (batch,))."""
    if not _is_device_tensor(rows):
        raise N.InvalidArgument("rdo_select_batch takes device rows; use rdo_select for one host signal")
    x, single = _dev_rows(rows, plan.size(), "rdo_select")
    b = x.shape[0]
    index = torch.empty((b,), dtype=torch.int32, device=x.device)
    chosen = torch.empty((b, plan.size()), dtype=x.dtype, device=x.device)
    pruned = torch.empty((b,), dtype=torch.uint8, device=x.device)
    fn = lib.dctp_ensemble_rdo_select_f64 if x.dtype == torch.float64 else lib.dctp_ensemble_rdo_select_f32
    stream = _stream_ptr(x.device)
    check(fn(plan._h, C.c_void_p(x.data_ptr()), C.c_void_p(chosen.data_ptr()), C.c_void_p(index.data_ptr()),
             C.c_void_p(pruned.data_ptr()), b, stream))
    if sync:
        check(lib.dctp_ensemble_sync_check(plan._h, stream))
    return (index[0], chosen[0], pruned[0]) if single else (index, chosen, pruned)


def calibrate_prune_threshold(n: int, r: float = 0.99, quantile: float = 0.7, trials: int = 512,
                              seed: int = 42) -> float:
    """bench.hpp:99-108: the `quantile` of the path quadratic form over
    `trials` AR(r) signals drawn from Rng(mix_seed(seed, n, 9000))."""
    sig = fill_signals(mix_seed(seed, n, 9000), DIST_AR, n, trials, r)
    d = sig[:, :-1] - sig[:, 1:]
    q = np.sort(np.cumsum(d * d, axis=1)[:, -1])  # sequential sums, as the reference
    return float(q[min(trials - 1, int(quantile * (trials - 1)))])


# --- batched trig kernels (trig.hpp:95-110) -------------------------------------------

# --- rank-k chains (cauchy.hpp:159-231) ---------------------------------------


class SpectralBasis:
    """L = U diag(lambda) U^T, lambda ascending, column k of u = eigenvector k
    (spectral.hpp:21-24)."""

    def __init__(self, lambda_, u):
        self.lambda_ = np.ascontiguousarray(np.asarray(lambda_, dtype=np.float64))
        self.u = np.ascontiguousarray(np.asarray(u, dtype=np.float64))
        n = self.lambda_.shape[0]
        if self.lambda_.ndim != 1 or self.u.shape != (n, n):
            raise N.InvalidArgument("SpectralBasis: lambda (n,) and u (n, n) expected")


def path_spectrum(n: int) -> SpectralBasis:
    """Unit-weight path graph (spectral.hpp:48-68): the base of every plan."""
    if n < 2:
        raise N.InvalidArgument("path_spectrum: need n >= 2")
    lam = 2.0 - 2.0 * np.cos(np.arange(n) * np.pi / n)
    lam[0] = 0.0
    k, j = np.meshgrid(np.arange(n), np.arange(n))
    u = np.sqrt(2.0 / n) * np.cos(np.pi * k * (2.0 * j + 1.0) / (2.0 * n))
    u[:, 0] /= np.sqrt(2.0)
    b = SpectralBasis(lam, u)
    b._path = True  # compose_rank_k rebuilds it on the host with the reference's rounding
    return b


class ChainedFactorization:
    """compose_rank_k(base, updates, tau) (cauchy.hpp:163-216): k rank-one
    updates applied in order.  The composition runs on the host (the final
    basis x and eigenvalues mu match the reference bit for bit); chain_forward
    runs on the GPU as one product with x."""

    def __init__(self, base, updates: Sequence[RankOneUpdate], tau: float = 1e-12, device: int = 0):
        if isinstance(base, (int, np.integer)):
            base = path_spectrum(int(base))
        n = base.lambda_.shape[0]
        k = len(updates)
        kinds = (C.c_int * max(k, 1))(*[u.kind for u in updates])
        is_ = (C.c_size_t * max(k, 1))(*[u.node_i for u in updates])
        js = (C.c_size_t * max(k, 1))(*[u.node_j for u in updates])
        rhos = (C.c_double * max(k, 1))(*[u.rho for u in updates])
        vs = None
        if any(u.kind == GENERAL for u in updates):
            vs = np.zeros((k, n))
            for r, u in enumerate(updates):
                if u.kind == GENERAL:
                    if np.asarray(u.v).shape[0] != n:
                        raise N.RuntimeFailure(f"compose_rank_k: stage {r + 1}: RankOneUpdate: direction length "
                                               "mismatch")
                    vs[r] = u.direction(n)
        path = getattr(base, "_path", False)
        bl = None if path else base.lambda_.ctypes.data_as(C.c_void_p)
        bu = None if path else base.u.ctypes.data_as(C.c_void_p)
        h = C.c_void_p()
        check(lib.dctp_chain_create(n, k, kinds, is_, js, rhos, None if vs is None else vs.ctypes.data_as(C.c_void_p),
                                    bl, bu, float(tau), int(device), C.byref(h)))
        self._h = h
        self.n, self.device, self.updates = n, device, list(updates)
        self.base = base
        mu, x = np.empty(n), np.empty((n, n))
        check(lib.dctp_chain_spectrum(h, mu.ctypes.data_as(C.c_void_p), x.ctypes.data_as(C.c_void_p)))
        self.mu, self.x = mu, x

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and lib is not None:
            lib.dctp_chain_destroy(h)
            self._h = None

    @property
    def stages(self) -> list:
        """Per stage: base_vals, mu, sigma, slot map, rotation count (ChainStage)."""
        out = []
        for r in range(len(self.updates)):
            d = {k: np.empty(self.n) for k in ("base_vals", "mu", "sigma")}
            d["slot_pass"] = np.empty(self.n, dtype=np.int32)
            d["slot_idx"] = np.empty(self.n, dtype=np.int64)
            rot = C.c_size_t()
            check(lib.dctp_chain_stage(self._h, r, *[d[k].ctypes.data_as(C.c_void_p) for k in
                                                     ("base_vals", "mu", "sigma", "slot_pass", "slot_idx")],
                                       C.byref(rot)))
            d["rotations"] = rot.value
            out.append(d)
        return out

    def forward(self, s, sync: bool = True, out=None):
        """chain_forward (cauchy.hpp:218-231) for one signal or a batch of rows."""
        n = self.n
        if _is_device_tensor(s):
            rows, single = _dev_rows(s, n, "chain_forward")
            y = _check_out(out, rows, rows.shape, "chain_forward") if out is not None else torch.empty_like(rows)
            fn = lib.dctp_chain_forward_f64 if rows.dtype == torch.float64 else lib.dctp_chain_forward_f32
            stream = _stream_ptr(rows.device)
            check(fn(self._h, C.c_void_p(rows.data_ptr()), C.c_void_p(y.data_ptr()), rows.shape[0], stream))
            if sync:
                check(lib.dctp_chain_sync_check(self._h, stream))
            return y.reshape(-1) if single else y
        rows, single = _as_rows(s, n, "chain_forward")
        y = np.empty_like(rows)
        fn = lib.dctp_chain_forward_host_f64 if rows.dtype == np.float64 else lib.dctp_chain_forward_host_f32
        check(fn(self._h, rows.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), rows.shape[0]))
        return y.reshape(-1) if single else y

    def sync_check(self):
        check(lib.dctp_chain_sync_check(self._h, _stream_ptr(torch.cuda.current_device())))


def compose_rank_k(base, updates: Sequence[RankOneUpdate], tau: float = 1e-12, device: int = 0
                   ) -> ChainedFactorization:
    return ChainedFactorization(base, updates, tau, device)


def chain_forward(chain: ChainedFactorization, s):
    return chain.forward(s)


def _trig(x, inverse: bool):
    if not _is_device_tensor(x):
        raise N.InvalidArgument("dct2/idct2 batch kernels take CUDA tensors")
    rows = x.reshape(1, -1) if x.dim() == 1 else x
    rows = rows.contiguous()
    n = rows.shape[1]
    y = torch.empty_like(rows)
    fn = {(False, True): lib.dctp_dct2_f64, (False, False): lib.dctp_dct2_f32,
          (True, True): lib.dctp_idct2_f64, (True, False): lib.dctp_idct2_f32}[(inverse, rows.dtype == torch.float64)]
    check(fn(n, C.c_void_p(rows.data_ptr()), C.c_void_p(y.data_ptr()), rows.shape[0], rows.device.index,
             _stream_ptr(rows.device)))
    return y.reshape(x.shape)


def dct2(x):
    """Orthonormal DCT-II (U^T s) of each row on the GPU."""
    return _trig(x, False)


def idct2(x):
    """Inverse of dct2 (U p) of each row on the GPU."""
    return _trig(x, True)


# --- seeded inputs (signal.hpp / bench.hpp) -------------------------------------------

DIST_GAUSSIAN, DIST_UNIFORM, DIST_AR, DIST_SYM_UNIFORM, DIST_AR2D = 0, 1, 2, 3, 4


def mix_seed(seed: int, size: int, kind: int) -> int:
    return int(lib.dctp_mix_seed(seed, size, kind))


def fill_signals(seed: int, dist: int, n: int, rows: int, r: float = 0.0) -> np.ndarray:
    """rows x n samples from Rng(seed) (signal.hpp:18-55): 0 gaussian, 1 uniform,
    2 gen_ar_signal(n, r) rows, 3 2*uniform-1, 4 2-D separable AR(1) rows."""
    out = np.empty((rows, n))
    check(lib.dctp_fill_signals(seed, dist, float(r), n, rows, out.ctypes.data_as(C.c_void_p)))
    return out


def ozaki_slices(n: int) -> int:
    """int8 digits per operand the fp64 dense products of length-n rows use on
    the tcgen05 kind::i8 path (0: the DMMA fp64 tensor cores) — dctp_ozaki_slices."""
    s = C.c_int()
    check(lib.dctp_ozaki_slices(int(n), C.byref(s)))
    return s.value


# --- kernel profiling (CUDA events around every launch; bench.py) ---------------------

def profile_enable(on: bool = True) -> None:
    check(lib.dctp_profile_enable(1 if on else 0))


def profile_reset() -> None:
    check(lib.dctp_profile_reset())


def profile_summary() -> dict:
    """{kernel: (launches, total_ms)} since the last reset (waits for the events)."""
    import json

    buf = C.create_string_buffer(1 << 16)
    check(lib.dctp_profile_summary(buf, len(buf)))
    return {k: (int(v[0]), float(v[1])) for k, v in json.loads(buf.value.decode()).items()}
