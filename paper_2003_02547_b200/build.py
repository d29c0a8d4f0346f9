"""In-tree build of the CUDA library (nvcc, sm_100a) -- no JIT caches.

``python -m paper_2003_02547_b200.build [--force] [-v]`` compiles every
``csrc/*.cu`` to an object in ``build/`` (in parallel) and links
``paper_2003_02547_b200/_lib/libocpqp_b200.so`` (static cudart, the C ABI of
include/ocpqp_b200.h).  Only sources newer than their object are rebuilt.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
OUT = PKG / "_lib" / "libocpqp_b200.so"
HEADERS = [CSRC / "ocpqp_internal.h", CSRC / "ocpqp_fast.cuh", CSRC / "ocpqp_row.cuh",
           ROOT / "include" / "ocpqp_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
] + os.environ.get("OCPQP_NVCC_EXTRA", "").split()


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    return "nvcc"


def sources():
    return sorted(CSRC.glob("*.cu"))


def _stale(src, obj):
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return src.stat().st_mtime > t or any(h.stat().st_mtime > t for h in HEADERS if h.exists())


def build(force=False, verbose=False, jobs=None):
    OBJ.mkdir(parents=True, exist_ok=True)
    OUT.parent.mkdir(parents=True, exist_ok=True)
    srcs = sources()
    objs = [OBJ / (s.stem + ".o") for s in srcs]
    todo = [(s, o) for s, o in zip(srcs, objs) if force or _stale(s, o)]

    def compile_one(so):
        s, o = so
        cmd = [nvcc(), *NVCC_FLAGS, "-c", str(s), "-o", str(o)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {s.name}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return o

    if todo:
        with ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
            list(ex.map(compile_one, todo))
    if todo or not OUT.exists() or any(o.stat().st_mtime > OUT.stat().st_mtime for o in objs):
        cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart",
               "static", "-o", str(OUT), *map(str, objs)]
        subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
