"""The warp-specialized DMMA kernels off the round-1 fast path (VERDICT r1
"performance cliff"): b_a = 64 and non-power-of-two (even and odd) b_c,
against the numpy oracle (pinned to the reference's golden vectors) in every
execution mode - device run, pipelined host run, pageable host run,
reuse=False - at relative Frobenius 1e-12."""

import numpy as np
import pytest

import paper_1301_7744_b200 as bs
from oracle import bcss_oracle as orc

pytestmark = pytest.mark.gpu

CASES = [
    (3, 128, 128, 64, 64), (2, 192, 128, 64, 32), (3, 128, 96, 64, 48), (4, 64, 64, 64, 16),
    (3, 96, 96, 32, 6), (4, 64, 60, 16, 12), (4, 32, 30, 8, 3), (3, 64, 45, 32, 5),
    (5, 16, 24, 8, 6), (3, 32, 36, 4, 12),
]


@pytest.mark.parametrize("cfg", CASES, ids=lambda c: "m%d_n%d_p%d_ba%d_bc%d" % c)
def test_fast_kernels_match_oracle(cfg, kernels):
    import torch

    m, n, p, ba, bc = cfg
    rng = np.random.default_rng(sum(cfg))
    a = orc.random_bcss_packed(m, n, ba, int(rng.integers(1 << 30)))
    x = rng.standard_normal((p, n))
    want = orc.sttsm_bcss_packed(a, x, m, n, ba, bc)
    plan = bs.SttsmPlan(m, n, p, ba, bc)
    if kernels == "fast" or (m > 2 and ba ** (m - 1) >= 64):
        assert plan.stats()["generic_launches"] == 0
    c = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64, device="cuda")
    plan.run(torch.from_numpy(a).cuda(), torch.from_numpy(x).cuda(), c)
    torch.cuda.synchronize()
    assert orc.rel_frobenius(c.cpu().numpy(), want) <= 1e-12
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
