"""In-tree build of the CUDA extension (sm_100a) -> paper_2409_07232_b200/_lib/libfsbm_coal.so.

Plain nvcc, no torch extension machinery: the product is a C-ABI shared library
(include/fsbm_coal.h).  The .so is git-ignored but travels to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
SO = os.path.join(OUT_DIR, "libfsbm_coal.so")
SOURCES = ["fsbm_coal.cu"]
HEADERS = ["fsbm_common.cuh", "coal_exact.cuh", "coal_fast.cuh", "coal_dmma.cuh", "coal_dmmag.cuh", "coal_bott.cuh", "state_io.cuh", "fsbm_group.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
         "-Xptxas", "-v", "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "fsbm_coal.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return SO
    os.makedirs(OUT_DIR, exist_ok=True)
    cmd = [NVCC] + ARCH + FLAGS + [os.path.join(CSRC, f) for f in SOURCES] + ["-o", SO + ".tmp", "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(OUT_DIR, "build.log")
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-8000:])
        raise RuntimeError(f"nvcc failed ({res.returncode}); see {log}")
    os.replace(SO + ".tmp", SO)
    if verbose:
        sys.stdout.write(res.stderr)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(SO)
