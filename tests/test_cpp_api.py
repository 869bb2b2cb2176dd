"""The C++ mirror header compiles against the C ABI (CPU) and its test
program passes on the GPU (tests/cpp/test_cpp_api.cpp)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIBDIR = ROOT / "paper_2409_08970_b200" / "lib"
EXE = ROOT / "paper_2409_08970_b200" / "build" / "test_cpp_api"


def build_exe():
    EXE.parent.mkdir(parents=True, exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", str(ROOT / "include"), "-I", "/usr/local/cuda/include",
           str(ROOT / "tests" / "cpp" / "test_cpp_api.cpp"), "-o", str(EXE), "-L", str(LIBDIR), "-ldctplus_b200",
           f"-Wl,-rpath,{LIBDIR}", "-L", "/usr/local/cuda/lib64", "-lcudart"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_cpp_mirror_compiles_and_links():
    build_exe()
    assert EXE.exists()


@pytest.mark.gpu
def test_cpp_mirror_api_on_gpu():
    build_exe()
    out = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ALL OK" in out.stdout, out.stdout + out.stderr
