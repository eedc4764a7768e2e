"""Build libmonet_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2010_14501_b200.build [--force] [--debug]

The shared library is the C-ABI of include/monet_b200.h; it is loaded with
ctypes (``_native.py``), so no torch headers are involved and the same .so
serves the Python executor, the tests and a foreign (cgo/JNI/ctypes) host.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = PKG / "libmonet_b200.so"
DEBUG_LIB = PKG / "libmonet_b200_dbg.so"  # + GEMM operand-dump / wait-counter hooks (tools/ only)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

CU_SOURCES = ["capi.cu", "profile.cu", "comm.cu"]
CPP_SOURCES = ["arena.cpp", "bnb.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    files = [CSRC / f for f in CU_SOURCES + CPP_SOURCES]
    files += list(CSRC.glob("*.cuh")) + [INCLUDE / "monet_b200.h", CSRC / "exports.map"]
    return files


def needs_build(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    return any(f.stat().st_mtime > t for f in _sources())


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> Path:
    lib = DEBUG_LIB if debug else LIB
    if not force and not needs_build(lib):
        return lib
    out_dir = PKG / ("build_dbg" if debug else "build")
    out_dir.mkdir(exist_ok=True)
    objs = []
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", str(INCLUDE)] + (["-DMONET_DEBUG"] if debug else [])
    for src in CU_SOURCES:
        obj = out_dir / (src + ".o")
        cmd = [NVCC, *ARCH, "-lineinfo", *common, "--expt-relaxed-constexpr", "-Xptxas", "-v",
               "-c", str(CSRC / src), "-o", str(obj)]
        _run(cmd, verbose)
        objs.append(obj)
    for src in CPP_SOURCES:
        obj = out_dir / (src + ".o")
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-I", str(INCLUDE), "-c", str(CSRC / src),
              "-o", str(obj)], verbose)
        objs.append(obj)
    tmp = lib.with_suffix(".so.tmp")
    # export only the extern "C" monet_* boundary (exports.map)
    _run([NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart", "-ldl",
          "-Xlinker", f"--version-script={CSRC / 'exports.map'}"], verbose)
    os.replace(tmp, lib)
    return lib


def _run(cmd, verbose):
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode:
        sys.stderr.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode:
        raise RuntimeError(f"build step failed: {cmd[0]} (exit {res.returncode})")
    (PKG / "build").mkdir(exist_ok=True)
    (PKG / "build" / "ptxas.log").open("a").write(res.stderr)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv))
