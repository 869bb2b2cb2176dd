"""The C-ABI library loads and exports every symbol include/dctplus_b200.h
declares (CPU; no compute calls)."""
import ctypes
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "dctplus_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dctp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("dctp_plan_create", "dctp_forward_f64", "dctp_inverse_f32", "dctp_ensemble_forward_all_f32",
                 "dctp_plan_sync_check", "dctp_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2409_08970_b200 import _native

    lib = ctypes.CDLL(str(_native.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared_symbols()) == set(_native.SIGNATURES), "ctypes binding drifted from the header"


def test_library_is_sm100a_device_code():
    from paper_2409_08970_b200 import _native

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out, out


def test_version_and_error_channel():
    from paper_2409_08970_b200 import _native

    assert b"sm_100a" in _native.lib.dctp_version()
    h = ctypes.c_void_p()
    rc = _native.lib.dctp_plan_create(1, 0, 1, 0, 1.0, None, 1e-12, 1e-12, -1, ctypes.byref(h))
    assert rc == 1 and b"n >= 2" in _native.lib.dctp_last_error()
