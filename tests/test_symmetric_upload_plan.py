"""Host side of the symmetric upload (csrc/sym_upload.cu), no GPU needed:
the bytes a plan reports moving equal a brute-force count of the sectors that
hold orbit representatives, and every element left out is filled from a
representative that was uploaded."""

import itertools

import pytest

import paper_1301_7744_b200 as bs
from oracle import bcss_oracle as orc


def _runs(key):
    return [d for d in range(1, len(key)) if key[d] == key[d - 1]]


def _fetched(dig, runs):
    # the kernel's predicate: mode 0 by 4-double sectors, other modes exactly
    ok = True
    for d in runs:
        if d == 1:
            ok &= (dig[0] >> 2) <= (dig[1] >> 2)
        else:
            ok &= dig[d - 1] <= dig[d]
    return ok


def _rep(dig, runs):
    v = list(dig)
    for _ in range(len(v)):
        for d in runs:
            if v[d - 1] > v[d]:
                v[d - 1], v[d] = v[d], v[d - 1]
    return tuple(v)


@pytest.mark.parametrize("cfg", [(3, 16, 4), (2, 32, 8), (4, 16, 8), (3, 64, 16), (5, 8, 4), (4, 12, 4)])
def test_upload_bytes_match_brute_force(cfg):
    m, n, b = cfg
    plan = bs.SttsmPlan(m, n, n, b, b, pipeline=2, symmetric_upload=True)
    total = 0
    for key in orc.hypertriangle(n // b, m):
        runs = _runs(key)
        if not runs:
            total += b**m
            continue
        for dig in itertools.product(range(b), repeat=m):
            if _fetched(dig, runs):
                total += 1
            else:
                assert _fetched(_rep(dig, runs), runs)  # filled from an uploaded element
    assert plan.upload_bytes == 8 * total < 8 * plan.a_elems
    plan.close()


def test_upload_bytes_without_symmetric_upload():
    for kw in ({}, {"symmetric_upload": True}):
        # non-pipelined plans and b_a < 4 / non-powers of two move all of A
        for cfg, pipe in (((3, 16, 16, 4, 4), 0), ((3, 12, 12, 3, 3), 2), ((3, 16, 16, 2, 2), 2)):
            plan = bs.SttsmPlan(*cfg, pipeline=pipe, **kw)
            assert plan.upload_bytes == 8 * plan.a_elems
            plan.close()
    plan = bs.SttsmPlan(3, 16, 16, 4, 4, pipeline=2)
    assert plan.upload_bytes == 8 * plan.a_elems and plan.last_upload_bytes == -1
    plan.close()


def test_baseline_config_fractions():
    # the fraction of A each BASELINE config moves over PCIe
    want = {(4, 512, 256, 32, 32): 0.7211, (3, 512, 512, 32, 32): 0.8489,
            (4, 192, 192, 16, 16): 0.6733, (5, 96, 96, 8, 8): 0.5668}
    for cfg, frac in want.items():
        plan = bs.SttsmPlan(*cfg, pipeline=4, symmetric_upload=True)
        assert abs(plan.upload_bytes / (8 * plan.a_elems) - frac) < 1e-4
        plan.close()
