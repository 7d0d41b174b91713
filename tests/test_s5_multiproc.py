"""S5 with 8 ranks (8 processes sharing the one GPU): owners, two helpers
(T(m-1) peer copies), fused T(m-2) peer stores into every assignee's slots,
subtree groups gated on other processes' CUDA IPC events, gloo host barriers,
three steps - the assembled C equals the single-plan C bit for bit
(tools/s5_multiproc_check.py)."""
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.gpu
def test_s5_eight_processes_with_helpers_bitwise():
    res = subprocess.run([sys.executable, "tools/s5_multiproc_check.py", "8", "4", "256", "128", "16", "16"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert '"bitwise_equal": true' in res.stdout and '"helpers": {}' not in res.stdout
