"""In-tree build of the native library (sm_100a CUDA kernels + C++ host).

Output: paper_2409_08970_b200/lib/libdctplus_b200.so (git-ignored; travels to
the GPU box with gpurun).  Kernels: nvcc -gencode arch=compute_100a,code=sm_100a
-lineinfo.  Host setup: g++ -std=c++20 -ffp-contract=off (the per-graph setup
must reproduce the reference's floating-point operations bit for bit).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "build"
LIB = PKG / "lib" / "libdctplus_b200.so"

CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SOURCES = sorted((CSRC / "kernels").glob("*.cu"))
CPP_SOURCES = [CSRC / "capi.cpp"]
HEADERS = (
    sorted(CSRC.rglob("*.hpp")) + sorted(CSRC.rglob("*.cuh")) + sorted((ROOT / "include").rglob("*.h"))
)

INCLUDES = ["-I", str(CSRC), "-I", str(ROOT / "include")]

# setup.cu restates the host setup's floating-point operations one for one:
# no multiply-add contraction, so its roots are bit-identical to the host's.
FILE_FLAGS = {"setup.cu": ["-fmad=false"]}


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    LIB.parent.mkdir(parents=True, exist_ok=True)
    objs = []
    for src in CU_SOURCES:
        obj = BUILD / (src.stem + ".cu.o")
        if force or _stale(obj, [src, *HEADERS, __file__]):
            _run([NVCC, "-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC",
                  "-Xptxas", "-warn-spills", "--expt-relaxed-constexpr", *FILE_FLAGS.get(src.name, []), *INCLUDES,
                  "-c", str(src), "-o", str(obj)], verbose)
        objs.append(obj)
    for src in CPP_SOURCES:
        obj = BUILD / (src.stem + ".cpp.o")
        if force or _stale(obj, [src, *HEADERS, __file__]):
            _run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-Wall", "-Wno-unused-function",
                  *INCLUDES, "-I", str(CUDA_HOME / "include"), "-c", str(src), "-o", str(obj)], verbose)
        objs.append(obj)
    if force or _stale(LIB, objs):
        tmp = LIB.with_suffix(".so.tmp")
        _run([NVCC, "-shared", *ARCH, "-Xcompiler", "-fPIC", *map(str, objs), "-o", str(tmp),
              "-lpthread", "-ldl", "-lrt"], verbose)
        shutil.move(str(tmp), str(LIB))
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
    print(LIB)
