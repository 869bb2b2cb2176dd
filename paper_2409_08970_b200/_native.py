"""ctypes binding of the C ABI in include/dctplus_b200.h.

The shared library is built in-tree (paper_2409_08970_b200/lib/) by
``paper_2409_08970_b200._build.build()``.  There is no fallback: if the
library is missing or fails to load, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libdctplus_b200.so"

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback for the DCT+ path)"
    )

lib = C.CDLL(str(LIB_PATH))

_sz = C.c_size_t
_p = C.c_void_p
_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int)

# name -> (restype, argtypes); every symbol include/dctplus_b200.h declares.
SIGNATURES = {
    "dctp_last_error": (C.c_char_p, []),
    "dctp_version": (C.c_char_p, []),
    "dctp_plan_create": (C.c_int, [_sz, C.c_int, _sz, _sz, C.c_double, _p, C.c_double, C.c_double, C.c_int,
                                    C.POINTER(_p)]),
    "dctp_plan_destroy": (C.c_int, [_p]),
    "dctp_plan_info": (C.c_int, [_p, C.POINTER(_sz), _dp, _ip, C.POINTER(_sz), C.POINTER(_sz), _ip]),
    "dctp_plan_route": (C.c_int, [_p, _ip, _dp]),
    "dctp_ozaki_slices": (C.c_int, [_sz, _ip]),
    "dctp_plan_setup": (C.c_int, [_p, _p, _p, _p, _p, _p]),
    "dctp_plan_slots": (C.c_int, [_p, _p, _p]),
    "dctp_plan_subproblem": (C.c_int, [_p, C.POINTER(_sz), _p, _p, _p, _dp]),
    "dctp_plan_basis": (C.c_int, [_p, _p]),
    "dctp_forward_f64": (C.c_int, [_p, _p, _p, _sz, _p]),
    "dctp_forward_f32": (C.c_int, [_p, _p, _p, _sz, _p]),
    "dctp_inverse_f64": (C.c_int, [_p, _p, _p, _sz, _p]),
    "dctp_inverse_f32": (C.c_int, [_p, _p, _p, _sz, _p]),
    "dctp_plan_sync_check": (C.c_int, [_p, _p]),
    "dctp_forward_nmvp_f64": (C.c_int, [_p, _p, _p, _sz, _p]),
    "dctp_forward_nmvp_f32": (C.c_int, [_p, _p, _p, _sz, _p]),
    "dctp_inverse_nmvp_f64": (C.c_int, [_p, _p, _p, _sz, _p]),
    "dctp_inverse_nmvp_f32": (C.c_int, [_p, _p, _p, _sz, _p]),
    "dctp_forward_nmvp_host_f64": (C.c_int, [_p, _p, _p, _sz]),
    "dctp_forward_nmvp_host_f32": (C.c_int, [_p, _p, _p, _sz]),
    "dctp_inverse_nmvp_host_f64": (C.c_int, [_p, _p, _p, _sz]),
    "dctp_inverse_nmvp_host_f32": (C.c_int, [_p, _p, _p, _sz]),
    "dctp_forward_host_f64": (C.c_int, [_p, _p, _p, _sz]),
    "dctp_inverse_host_f64": (C.c_int, [_p, _p, _p, _sz]),
    "dctp_forward_host_f32": (C.c_int, [_p, _p, _p, _sz]),
    "dctp_inverse_host_f32": (C.c_int, [_p, _p, _p, _sz]),
    "dctp_ensemble_create": (C.c_int, [_sz, _sz, _p, _p, _p, _p, _p, _sz, C.c_double, C.c_double, C.c_int,
                                        C.POINTER(_p)]),
    "dctp_ensemble_destroy": (C.c_int, [_p]),
    "dctp_ensemble_info": (C.c_int, [_p, C.POINTER(_sz), C.POINTER(_sz)]),
    "dctp_ensemble_member": (C.c_int, [_p, _sz, C.POINTER(_p)]),
    "dctp_ensemble_forward_all_f64": (C.c_int, [_p, _p, _p, _sz, _p]),
    "dctp_ensemble_forward_all_f32": (C.c_int, [_p, _p, _p, _sz, _p]),
    "dctp_ensemble_sync_check": (C.c_int, [_p, _p]),
    "dctp_ensemble_forward_all_pruned_f64": (C.c_int, [_p, _p, _p, _p, _p, _sz, _p]),
    "dctp_ensemble_forward_all_pruned_f32": (C.c_int, [_p, _p, _p, _p, _p, _sz, _p]),
    "dctp_ensemble_rdo_select_f64": (C.c_int, [_p, _p, _p, _p, _p, _sz, _p]),
    "dctp_ensemble_rdo_select_f32": (C.c_int, [_p, _p, _p, _p, _p, _sz, _p]),
    "dctp_ensemble_forward_all_pruned_host_f64": (C.c_int, [_p, _p, _p, _p, _p, _sz]),
    "dctp_ensemble_forward_all_pruned_host_f32": (C.c_int, [_p, _p, _p, _p, _p, _sz]),
    "dctp_ensemble_forward_all_host_f32": (C.c_int, [_p, _p, _p, _sz]),
    "dctp_ensemble_forward_all_host_f64": (C.c_int, [_p, _p, _p, _sz]),
    "dctp_chain_create": (C.c_int, [_sz, _sz, _p, _p, _p, _p, _p, _p, _p, C.c_double, C.c_int, C.POINTER(_p)]),
    "dctp_chain_destroy": (C.c_int, [_p]),
    "dctp_chain_info": (C.c_int, [_p, C.POINTER(_sz), C.POINTER(_sz)]),
    "dctp_chain_spectrum": (C.c_int, [_p, _p, _p]),
    "dctp_chain_stage": (C.c_int, [_p, _sz, _p, _p, _p, _p, _p, C.POINTER(_sz)]),
    "dctp_chain_forward_f64": (C.c_int, [_p, _p, _p, _sz, _p]),
    "dctp_chain_forward_f32": (C.c_int, [_p, _p, _p, _sz, _p]),
    "dctp_chain_sync_check": (C.c_int, [_p, _p]),
    "dctp_chain_forward_host_f64": (C.c_int, [_p, _p, _p, _sz]),
    "dctp_chain_forward_host_f32": (C.c_int, [_p, _p, _p, _sz]),
    "dctp_dct2_f64": (C.c_int, [_sz, _p, _p, _sz, C.c_int, _p]),
    "dctp_idct2_f64": (C.c_int, [_sz, _p, _p, _sz, C.c_int, _p]),
    "dctp_dct2_f32": (C.c_int, [_sz, _p, _p, _sz, C.c_int, _p]),
    "dctp_trig_host_f64": (C.c_int, [C.c_int, _sz, _p, _p, _sz, C.c_int]),
    "dctp_idct2_f32": (C.c_int, [_sz, _p, _p, _sz, C.c_int, _p]),
    "dctp_profile_enable": (C.c_int, [C.c_int]),
    "dctp_profile_reset": (C.c_int, []),
    "dctp_profile_summary": (C.c_int, [C.c_char_p, _sz]),
    "dctp_mix_seed": (C.c_uint64, [C.c_uint64, _sz, _sz]),
    "dctp_fill_signals": (C.c_int, [C.c_uint64, C.c_int, C.c_double, _sz, _sz, _p]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


class DctPlusError(Exception):
    """Base of the errors raised through the C ABI."""


class InvalidArgument(DctPlusError, ValueError):
    """std::invalid_argument in the reference."""


class DomainError(DctPlusError, ArithmeticError):
    """std::domain_error in the reference (non-finite input, pole collision)."""


class RuntimeFailure(DctPlusError, RuntimeError):
    """std::runtime_error in the reference (secular non-convergence)."""


class LogicError(DctPlusError, RuntimeError):
    """std::logic_error in the reference (repeated path eigenvalues, member index)."""


class CudaFailure(DctPlusError, RuntimeError):
    """A CUDA call failed (no reference counterpart)."""


_STATUS = {1: InvalidArgument, 2: DomainError, 3: RuntimeFailure, 4: LogicError, 5: CudaFailure}


def check(status: int) -> None:
    if status != 0:
        msg = lib.dctp_last_error().decode(errors="replace")
        raise _STATUS.get(status, DctPlusError)(msg)
