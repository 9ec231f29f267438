"""In-tree build of libgdwd_b200.so for sm_100a (nvcc, no torch extension).

    python -m paper_2305_12019_b200.build

The library is plain C ABI (include/gdwd_b200.h) loaded with ctypes; the
built .so lives next to this file so it travels with the repo snapshot.
``-fmad=false`` keeps every elementwise expression rounded like numpy (the
streaming matvecs are HBM-bound, so FMA contraction buys nothing there; the
Gram uses explicit DMMA instructions and is unaffected).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
LIB = HERE / "libgdwd_b200.so"
SOURCES = ["gdwd.cu", "gram.cu", "ingest.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "-Xcompiler", "-fPIC,-O2,-pthread", "-shared", "-cudart", "shared",
]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [
        HERE.parent / "include" / "gdwd_b200.h"]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    cmd = [NVCC, *FLAGS, *[str(CSRC / s) for s in SOURCES], "-o", str(LIB)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=str(CSRC))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
