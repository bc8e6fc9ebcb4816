"""Build the native libraries in-tree (they travel to the GPU box with the
repo snapshot; nothing is installed into site-packages).

* ``_lib/libgdsw_host.so`` – host symbolic runtime (C++, no CUDA).
* ``_lib/libgdsw.so``      – the sm_100a CUDA kernels behind the C ABI in
  ``include/gdsw.h``.

``python -m paper_2304_04876_b200.build`` rebuilds whatever is stale.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
LIB = PKG / "_lib"
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

HOST_SRC = [CSRC / "host" / "gdsw_host.cpp"]
CUDA_SRC = [CSRC / "gdsw_abi.cu"]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _deps(*dirs, suffixes=(".cu", ".cuh", ".inc", ".cpp", ".h", ".hpp")):
    out = []
    for d in dirs:
        for p in Path(d).rglob("*"):
            if p.suffix in suffixes:
                out.append(p)
    return out


def _run(cmd):
    print("+", " ".join(str(c) for c in cmd), flush=True)
    subprocess.run([str(c) for c in cmd], check=True)


def build_host(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libgdsw_host.so"
    if force or _stale(out, HOST_SRC + _deps(INCLUDE)):
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off",
              "-I", INCLUDE, *HOST_SRC, "-o", out])
    return out


def build_cuda(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libgdsw.so"
    if force or _stale(out, _deps(CSRC, INCLUDE)):
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-ffp-contract=off", "-shared", "-Xptxas", "-v", "-I", INCLUDE, "-I", CSRC,
              *CUDA_SRC, "-o", out, "-lcudart", "-Xlinker", "-rpath,/usr/local/cuda/lib64"])
    return out


def build_all(force: bool = False) -> None:
    build_host(force)
    build_cuda(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
