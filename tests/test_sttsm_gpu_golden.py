"""GPU parity against the reference's own outputs (tests/golden, made by
oracle/gen_golden.py from blocksym.sttsm_bcss): every case runs through the
drop-in ``sttsm_bcss`` (C ABI -> sm_100a DMMA kernels) and must match the
reference within relative Frobenius 1e-12 (BASELINE north star) and the
reference tests' max-rel bar 1e-10 (test_change_of_basis.py:126-136)."""

import glob

import numpy as np
import pytest

import paper_1301_7744_b200 as bs
from oracle import bcss_oracle as orc

pytestmark = pytest.mark.gpu

CASES = sorted(glob.glob(str(__import__("conftest").GOLDEN / "sttsm_*.npz")))


def _load(path):
    d = np.load(path)
    m, n, p, b_a, b_c = (int(v) for v in d["dims"])
    return d, m, n, p, b_a, b_c


@pytest.mark.parametrize("path", CASES, ids=lambda s: s.split("/")[-1][6:-4])
@pytest.mark.parametrize("reuse", [True, False])
def test_drop_in_matches_reference(path, reuse, kernels):
    d, m, n, p, b_a, b_c = _load(path)
    a = bs.BcssTensor(m, n, b_a, payload=d["A"])
    ctr = bs.OpCounter()
    out = bs.sttsm_bcss(a, d["X"], b_c, ctr, reuse=reuse)
    want = d["C"] if reuse else d["C_noreuse"]
    assert out.dims == (p,) * m and out.b == b_c
    assert orc.rel_frobenius(out.payload, want) <= 1e-12
    assert orc.max_rel(out.payload, want) <= 1e-10
    if "C_naive" in d:
        assert orc.rel_frobenius(out.payload, d["C_naive"]) <= 1e-12
    assert ctr.flops == int(d["flops"][0 if reuse else 1])


def test_temp_hook_replays_reference_temporaries(golden_dir):
    d = np.load(golden_dir / "temps_m4_n4_b2.npz")
    a = bs.BcssTensor(4, 4, 2, payload=d["A"])
    seen = []
    bs.sttsm_bcss(a, d["X"], 2, temp_hook=lambda k, t: seen.append((k, t)))
    assert [k for k, _ in seen] == list(d["levels"])
    for i, (k, t) in enumerate(seen):
        assert orc.rel_frobenius(t.payload, d[f"T{i}"]) <= 1e-12
        assert t.dims == (4,) * k + (2,) * (4 - k)


@pytest.mark.parametrize("path", CASES, ids=lambda s: s.split("/")[-1][6:-4])
def test_pipelined_mirrored_plan_matches_reference(path, kernels):
    """The e2e path (pipelined plan: chunked upload, mirrored C order, per-wave
    downloads) on every golden case, through run_host with pinned buffers and
    through the device run."""
    import torch

    d, m, n, p, b_a, b_c = _load(path)
    plan = bs.SttsmPlan(m, n, p, b_a, b_c, pipeline=3)
    a_h = torch.from_numpy(np.ascontiguousarray(d["A"])).pin_memory()
    x_h = torch.from_numpy(np.ascontiguousarray(d["X"])).pin_memory()
    c_h = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64).pin_memory()
    plan.run_host(a_h.numpy(), x_h.numpy(), c_h.numpy())
    assert orc.rel_frobenius(c_h.numpy(), d["C"]) <= 1e-12
    assert orc.max_rel(c_h.numpy(), d["C"]) <= 1e-10
    c_d = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64, device="cuda")
    plan.run(a_h.cuda(), x_h.cuda(), c_d)
    torch.cuda.synchronize()
    assert torch.equal(c_d.cpu(), c_h)
    # pageable host buffers: the same plan falls back to serial copies
    c_p = np.full(plan.c_elems, np.nan)
    plan.run_host(np.ascontiguousarray(d["A"]), np.ascontiguousarray(d["X"]), c_p)
    assert np.array_equal(c_p, c_h.numpy())
    plan.close()
