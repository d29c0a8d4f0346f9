"""In-tree build of the CUDA library (nvcc, sm_100a) -- no JIT caches.

``python -m paper_2003_02547_b200.build`` produces
``paper_2003_02547_b200/_lib/libocpqp_b200.so`` (static cudart, C ABI of
include/ocpqp_b200.h).  Rebuilds only when a source is newer than the .so.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "_lib" / "libocpqp_b200.so"
SOURCES = [CSRC / "ocpqp_ipm.cu", CSRC / "ocpqp_capi.cu"]
DEPS = SOURCES + [CSRC / "ocpqp_internal.h", ROOT / "include" / "ocpqp_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    return "nvcc"


def needs_build():
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def build(force=False, verbose=False):
    if not force and not needs_build():
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    cmd = [nvcc(), *NVCC_FLAGS, "-o", str(OUT), *map(str, SOURCES)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
