"""Non-power-of-two b_a on the warp-specialized DMMA kernels (POW2 = false:
row groups of 4, 12, 20, 24 or 28 dividing b_a, runtime b_a^p addressing,
[e][col] staging, division epilogue) against the numpy oracle (pinned to the
reference's golden vectors) at relative Frobenius 1e-12, in every execution
mode that reaches them: device run, pipelined host run (mirrored level 0),
pageable host run, reuse=False below the top level, a forced-wave plan."""

import numpy as np
import pytest

import paper_1301_7744_b200 as bs
from oracle import bcss_oracle as orc

pytestmark = pytest.mark.gpu

CASES = [
    (3, 48, 40, 12, 8), (2, 72, 48, 24, 16), (3, 72, 64, 24, 32), (3, 60, 40, 20, 8), (3, 56, 32, 28, 16),
    (4, 36, 24, 12, 8), (3, 96, 64, 48, 16), (3, 88, 48, 44, 8), (4, 40, 24, 20, 12), (3, 72, 72, 36, 24),
    (2, 120, 60, 40, 20), (5, 24, 16, 12, 8),
    # b_a that no row group divides (odd ones included): the contraction runs
    # over blocks padded to b_a' rows (zero-filled), X over padded column blocks
    (3, 30, 24, 10, 8), (3, 42, 16, 14, 8), (2, 66, 32, 22, 16), (3, 45, 20, 15, 5), (3, 27, 18, 9, 6),
    (4, 20, 12, 5, 4), (3, 42, 12, 6, 4), (3, 35, 21, 7, 7), (3, 54, 16, 18, 8), (3, 60, 24, 30, 8),
    (3, 66, 16, 33, 8), (2, 52, 26, 13, 13), (3, 50, 16, 25, 8), (4, 22, 8, 11, 4), (3, 63, 24, 21, 12),
    (3, 52, 16, 26, 16), (3, 54, 32, 27, 8), (5, 18, 8, 6, 4), (4, 28, 16, 14, 8),
]


@pytest.mark.parametrize("cfg", CASES, ids=lambda c: "m%d_n%d_p%d_ba%d_bc%d" % c)
def test_np_fast_kernels_match_oracle(cfg, kernels):
    import torch

    m, n, p, ba, bc = cfg
    rng = np.random.default_rng(sum(cfg) * 7)
    a = orc.random_bcss_packed(m, n, ba, int(rng.integers(1 << 30)))
    x = rng.standard_normal((p, n))
    want = orc.sttsm_bcss_packed(a, x, m, n, ba, bc)
    plan = bs.SttsmPlan(m, n, p, ba, bc)
    st = plan.stats()
    # (small odd b_a, and padded b_a with fewer than 64 top-level columns per
    # key, stay on the generic kernel: faster there)
    if (ba % 2 == 0 or ba >= 15) and (kernels == "fast" or (m > 2 and ba ** (m - 1) >= 64)):
        assert st["generic_launches"] == 0 and st["fast_launches"] > 0
    c = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64, device="cuda")
    plan.run(torch.from_numpy(a).cuda(), torch.from_numpy(x).cuda(), c)
    torch.cuda.synchronize()
    assert orc.rel_frobenius(c.cpu().numpy(), want) <= 1e-12
    ws = plan.workspace_bytes
    plan.close()
    pipe = bs.SttsmPlan(m, n, p, ba, bc, pipeline=3)
    ch = torch.full((pipe.c_elems,), float("nan"), dtype=torch.float64).pin_memory()
    pipe.run_host(torch.from_numpy(a).pin_memory().numpy(), torch.from_numpy(x).pin_memory().numpy(), ch.numpy())
    assert orc.rel_frobenius(ch.numpy(), want) <= 1e-12
    cp = np.full(pipe.c_elems, np.nan)
    pipe.run_host(a, x, cp)
    assert orc.rel_frobenius(cp, want) <= 1e-12
    pipe.close()
    nr = bs.SttsmPlan(m, n, p, ba, bc, reuse=False)
    c2 = torch.full((nr.c_elems,), float("nan"), dtype=torch.float64, device="cuda")
    nr.run(torch.from_numpy(a).cuda(), torch.from_numpy(x).cuda(), c2)
    torch.cuda.synchronize()
    assert orc.rel_frobenius(c2.cpu().numpy(), want) <= 1e-12
    nr.close()
    if ws > 0 and p // bc > 1:
        try:
            wv = bs.SttsmPlan(m, n, p, ba, bc, workspace_limit=max(1, ws // 2))
            c3 = torch.full((wv.c_elems,), float("nan"), dtype=torch.float64, device="cuda")
            wv.run(torch.from_numpy(a).cuda(), torch.from_numpy(x).cuda(), c3)
        except MemoryError:
            return  # one top-level unit does not fit half the workspace
        torch.cuda.synchronize()
        assert orc.rel_frobenius(c3.cpu().numpy(), want) <= 1e-12
        wv.close()
