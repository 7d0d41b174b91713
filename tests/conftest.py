import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


@pytest.fixture(params=["auto", "fast"])
def kernels(request, monkeypatch):
    """Kernel choice of the plans a test builds: "auto" is the product's own
    rule (problems with fewer than 64 top-level GEMM columns per key, and every
    m = 2 problem, run on the generic kernel: faster there), "fast" keeps the
    warp-specialized DMMA kernels wherever they apply (BCSS_FORCE_FAST), so the
    small golden shapes keep covering them.  The drop-in's plan cache is
    cleared on both sides (its key does not include the switch)."""
    import paper_1301_7744_b200 as bs

    bs.clear_plan_cache()
    if request.param == "fast":
        monkeypatch.setenv("BCSS_FORCE_FAST", "1")
    else:
        monkeypatch.delenv("BCSS_FORCE_FAST", raising=False)
    yield request.param
    bs.clear_plan_cache()
