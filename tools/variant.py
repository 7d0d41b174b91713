"""Run a tool against a variant library: python tools/variant.py NAME tool.py args..."""
import runpy
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1301_7744_b200 import _native  # noqa: E402

name = sys.argv[1]
_native.LIB_PATH = Path(__file__).resolve().parent / f"_bcss_{name}.so"
sys.argv = sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
