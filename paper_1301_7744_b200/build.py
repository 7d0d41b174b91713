"""In-tree build of the CUDA library (nvcc, sm_100a only)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SO = PKG / "_bcss_sttsm.so"
SOURCES = [PKG / "csrc" / "bcss_capi.cu"]
DEPS = SOURCES + [PKG / "csrc" / "sttsm_kernels.cuh", PKG / "csrc" / "combinatorics.hpp",
                  ROOT / "include" / "bcss_sttsm.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC", "-cudart", "shared",
         "-Xlinker", "-rpath,/usr/local/cuda/lib64", "-I", str(ROOT / "include")]


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and SO.exists() and all(SO.stat().st_mtime >= d.stat().st_mtime for d in DEPS):
        return SO
    cmd = [NVCC, *FLAGS, "-o", str(SO), *map(str, SOURCES)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed ({res.returncode}): {' '.join(cmd)}")
    if verbose:
        sys.stderr.write(res.stderr)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
