"""Build an experimental variant of the library (dev tool).

usage: python tools/build_variant.py NAME -DFLAG[=V] ...
Compiles every unit with the extra flags into build/obj_NAME/ and links
tools/_bcss_NAME.so; load it with tools/variant.py (sets _native.LIB_PATH).
"""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1301_7744_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
obj_dir = B.ROOT / "build" / f"obj_{name}"
obj_dir.mkdir(parents=True, exist_ok=True)


def comp(u):
    uname, src, defs = u
    cmd = [B.NVCC, *B.CFLAGS, *defs, *flags, "-c", "-o", str(obj_dir / f"{uname}.o"), str(src)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)


with ThreadPoolExecutor(8) as ex:
    list(ex.map(comp, B.UNITS))
so = B.ROOT / "tools" / f"_bcss_{name}.so"
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "shared", "-Xlinker", "-rpath,/usr/local/cuda/lib64",
                "-o", str(so), *[str(obj_dir / f"{u[0]}.o") for u in B.UNITS]], check=True)
print(so)
