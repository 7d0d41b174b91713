"""In-tree build of the CUDA library (nvcc, sm_100a only).

Translation units compile in parallel (one per fast b_a, the generic kernel,
the C ABI) into build/, then link into paper_1301_7744_b200/_bcss_sttsm.so.
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
SO = PKG / "_bcss_sttsm.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
          "-I", str(ROOT / "include")]
UNITS = [("bcss_capi", CSRC / "bcss_capi.cu", []),
         ("plan", CSRC / "plan.cu", []),
         ("run", CSRC / "run.cu", []),
         ("kernels_generic", CSRC / "kernels_generic.cu", []),
         ("symmetrize", CSRC / "symmetrize.cu", []),
         ("sym_upload", CSRC / "sym_upload.cu", [])] + [
    (f"kernels_fast_ba{ba}", CSRC / "kernels_fast.cu", [f"-DBCSS_BA={ba}"]) for ba in (4, 8, 16, 32, 64)] + [
    (f"kernels_np_rg{rg}", CSRC / "kernels_np.cu", [f"-DBCSS_NP_RG={rg}"]) for rg in (4, 12, 20, 24, 28)] + [
    (f"kernels_npp_rg{rg}", CSRC / "kernels_np.cu", [f"-DBCSS_NP_RG={rg}", "-DBCSS_NP_PAD=1"]) for rg in (4, 8, 12, 16, 20, 24, 28)]
HEADERS = [CSRC / "plan.hpp", CSRC / "sttsm_kernels.cuh", CSRC / "sttsm_ws_kernel.cuh", CSRC / "kernel_table.cuh", CSRC / "combinatorics.hpp", CSRC / "shape_costs.hpp",
           ROOT / "include" / "bcss_sttsm.h"]


def _stale(target: Path, deps) -> bool:
    return not target.exists() or any(target.stat().st_mtime < d.stat().st_mtime for d in deps)


def _compile(unit) -> tuple[str, str]:
    name, src, defs = unit
    obj = OBJ / f"{name}.o"
    cmd = [NVCC, *CFLAGS, *defs, "-c", "-o", str(obj), str(src)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {name}:\n{res.stdout}{res.stderr}")
    return name, res.stderr


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    todo = [u for u in UNITS if force or _stale(OBJ / f"{u[0]}.o", [u[1], *HEADERS])]
    if todo:
        with ThreadPoolExecutor(max_workers=min(len(todo), os.cpu_count() or 4)) as ex:
            for name, log in ex.map(_compile, todo):
                if verbose:
                    sys.stderr.write(f"--- {name}\n{log}")
    objs = [OBJ / f"{u[0]}.o" for u in UNITS]
    if force or todo or _stale(SO, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "shared", "-Xlinker", "-rpath,/usr/local/cuda/lib64",
               "-o", str(SO), *map(str, objs)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}{res.stderr}")
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
