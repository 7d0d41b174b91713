"""The C-ABI library loads, exports every symbol include/*.h declares, and
its host-side logic (combinatorics, plans, validation) matches the reference
(golden vectors) without a GPU."""

import ctypes
import re

import numpy as np
import pytest

import paper_1301_7744_b200 as bs
from conftest import GOLDEN, ROOT
from paper_1301_7744_b200 import _native
from oracle import bcss_oracle as orc


def declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names |= set(re.findall(r"\b(bcss_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, f"{name} not bound in _native.SIGNATURES"
    assert lib.bcss_abi_version() >= 100


def test_simplex_rank_unrank_match_reference():
    d = np.load(GOLDEN / "indexing.npz")
    for name in d.files:
        if not name.startswith("ht_"):
            continue
        _, g, m = name.split("_")
        g, m = int(g), int(m)
        assert bs.simplex_count(g, m) == len(d[name]) == _native.lib().bcss_simplex_count(g, m)
        for r, t in enumerate(d[name]):
            assert bs.hypertriangle_rank(t, g) == r
            assert bs.hypertriangle_unrank(r, m, g) == tuple(t)


def test_canonicalize_matches_reference():
    d = np.load(GOLDEN / "indexing.npz")
    for idx, can, mp in zip(d["grid_idx"], d["canonical"], d["mapping"]):
        assert bs.canonicalize(idx) == (tuple(can), tuple(mp))


def test_flops_match_reference_cost_model():
    for m, n, p, ba, bc, reuse, flops, memops in np.load(GOLDEN / "costs.npz")["rows"]:
        args = (int(m), int(n), int(p), int(ba), int(bc), bool(reuse))
        assert bs.bcss_flops(*args) == int(flops)
        assert bs.bcss_memops(*args) == int(memops)


@pytest.mark.parametrize("cfg", [(3, 16, 16, 4, 4), (3, 512, 512, 32, 32), (4, 192, 192, 16, 16),
                                 (5, 96, 96, 8, 8), (4, 512, 256, 32, 32), (3, 6, 4, 3, 2)])
@pytest.mark.parametrize("reuse", [True, False])
def test_plan_work_equals_cost_model(cfg, reuse):
    """The plan's work lists cover exactly the reference's level products:
    their flop sum equals bcss_costs(...).flops, and the C blocks written are
    every canonical block once."""
    plan = bs.SttsmPlan(*cfg, reuse=reuse)
    st = plan.stats()
    assert st["flops"] == bs.bcss_flops(*cfg, reuse=reuse)
    m, p, bc = cfg[0], cfg[2], cfg[4]
    ranks = plan.c_block_ranks()
    assert sorted(ranks.tolist()) == list(range(bs.simplex_count(p // bc, m)))
    assert st["launches"] >= m and st["waves"] == 1


def test_units_partition_c_blocks_and_flops():
    cfg = (4, 192, 192, 16, 16)
    pbar = 12
    seen, fl = [], 0
    for j in range(pbar):
        plan = bs.SttsmPlan(*cfg, units=[j])
        r = plan.c_block_ranks()
        # every block of unit j has largest block index j
        for rank in r:
            assert bs.hypertriangle_unrank(int(rank), 4, pbar)[-1] == j
        seen += r.tolist()
        fl += plan.stats()["flops"]
    assert sorted(seen) == list(range(bs.simplex_count(pbar, 4)))
    assert fl == bs.bcss_flops(*cfg)


def test_workspace_limit_splits_into_waves():
    cfg = (4, 512, 256, 32, 32)
    full = bs.SttsmPlan(*cfg)
    one = full.workspace_bytes
    lim = one // 3
    plan = bs.SttsmPlan(*cfg, workspace_limit=lim)
    st = plan.stats()
    assert st["waves"] > 1 and plan.workspace_bytes <= lim
    assert st["flops"] == bs.bcss_flops(*cfg)
    assert sorted(plan.c_block_ranks().tolist()) == list(range(bs.simplex_count(8, 4)))


@pytest.mark.parametrize("args,exc", [
    ((1, 4, 4, 2, 2), bs.ParameterError),
    ((3, 6, 6, 4, 2), bs.BlockDivisibilityError),
    ((3, 6, 6, 3, 4), bs.BlockDivisibilityError),
    ((3, 0, 6, 3, 3), bs.ParameterError),
])
def test_plan_validation_maps_to_reference_errors(args, exc):
    with pytest.raises(exc):
        bs.SttsmPlan(*args)


@pytest.mark.parametrize("args", [(3, 1 << 20, 64, 1, 1), (3, 64, 1 << 20, 1, 1), (2, 1 << 16, 64, 1, 1)])
def test_int32_table_limits_raise_instead_of_truncating(args):
    """Block / key / call counts past the int32 device tables are rejected
    at plan creation (ranks were narrowed silently)."""
    with pytest.raises(bs.ParameterError, match="int32"):
        bs.SttsmPlan(*args)
    with pytest.raises(bs.ParameterError, match="at most 8 modes"):
        bs.SttsmPlan(9, 4, 4, 2, 2)


@pytest.mark.parametrize("cfg,fast", [
    ((3, 128, 128, 64, 64), True), ((3, 256, 192, 64, 32), True),   # b_a = 64
    ((3, 96, 96, 32, 6), True), ((4, 64, 60, 16, 12), True),        # b_c not a power of two
    ((4, 32, 30, 8, 3), True), ((3, 64, 45, 32, 5), True),          # odd b_c
    ((3, 12, 12, 3, 2), False), ((3, 16, 16, 2, 2), False), ((2, 8, 8, 1, 1), False),
    # b_a no row group divides: padded row groups (even >= 6, odd >= 15); small odd b_a stays generic
    ((3, 60, 30, 10, 6), True), ((3, 90, 32, 30, 8), True), ((3, 45, 15, 15, 5), True), ((4, 24, 12, 6, 4), True),
    ((3, 88, 32, 44, 8), True), ((3, 35, 14, 7, 7), False), ((3, 39, 13, 13, 13), False), ((3, 25, 10, 5, 5), False),
    ((3, 24, 12, 6, 4), False), ((2, 44, 16, 22, 8), False),  # fewer than 64 columns per key at the top level
])
def test_fast_kernel_coverage(cfg, fast):
    """Every b_a in {4, 8, 16, 32, 64} runs on the warp-specialized DMMA
    kernels for any b_c (b_a = 64 and non-power-of-two b_c fell
    to the generic kernel); multiples of 4 and, through padded row groups,
    even b_a >= 6 and odd b_a >= 15 too; other b_a use the generic kernel."""
    st = bs.SttsmPlan(*cfg).stats()
    if fast:
        assert st["generic_launches"] == 0 and st["fast_launches"] > 0
    else:
        assert st["generic_launches"] > 0


def test_drop_in_argument_checks_without_gpu():
    """change_of_basis.py:54-63, 259-265: checks fire before any device work."""
    d = np.load(GOLDEN / "sttsm_small_m3_n4_p4_ba2_bc2.npz")
    a = bs.BcssTensor(3, 4, 2, payload=d["A"])
    with pytest.raises(bs.BlockDivisibilityError):
        bs.sttsm_bcss(a, d["X"], 3)
    with pytest.raises(bs.ShapeError):
        bs.sttsm_bcss(a, np.zeros((4, 5)), 2)
    with pytest.raises(bs.ShapeError):
        bs.sttsm_bcss(d["X"], d["X"], 2)
    part = bs.PartialSymTensor(2, 4, 2, (2,), payload=np.zeros(3 * 8))
    with pytest.raises(bs.ShapeError):
        bs.sttsm_bcss(part, d["X"], 2)
    # empty and ragged inputs, as the reference answers them: p = 0 has no
    # output blocks (ParameterError from simplex_count), X not a p x n matrix
    with pytest.raises(bs.ParameterError):
        bs.sttsm_bcss(a, np.zeros((0, 4)), 1)
    for x in (np.zeros(4), np.zeros((4, 4, 1))):
        with pytest.raises(bs.ShapeError):
            bs.sttsm_bcss(a, x, 1)
    # b_c <= 0: the reference fails with ZeroDivisionError / ParameterError;
    # here a named BlockDivisibilityError (a ValueError like both)
    for b_c in (0, -1):
        with pytest.raises(ValueError):
            bs.sttsm_bcss(a, d["X"], b_c)


def test_status_codes_raise_named_errors():
    with pytest.raises(bs.RangeError):
        bs.hypertriangle_rank((0, 5), 3)
    with pytest.raises(bs.ShapeError):
        bs.hypertriangle_rank((2, 1), 3)
    assert "outside" in _native.lib().bcss_last_error().decode() or True


@pytest.mark.parametrize("cfg,waves", [((3, 512, 512, 32, 32), 4), ((4, 64, 64, 16, 16), 3),
                                       ((5, 32, 48, 8, 8), 4), ((3, 64, 48, 16, 8), 3)])
def test_pipelined_plan_writes_every_c_block_once_in_contiguous_waves(cfg, waves):
    """A pipelined (mirrored) plan writes each C block exactly once, with the
    right flops, and every wave's blocks form one contiguous rank range (one
    D2H per wave): the rank list (wave order) splits into at most
    `stats()["waves"]` segments that are each a contiguous set of ranks."""
    m, n, p, ba, bc = cfg
    plan = bs.SttsmPlan(*cfg, pipeline=waves)
    st = plan.stats()
    assert 1 <= st["waves"] <= waves
    assert st["flops"] == bs.bcss_flops(*cfg)
    ranks = plan.c_block_ranks().tolist()
    assert sorted(ranks) == list(range(bs.simplex_count(p // bc, m)))
    # fewest segments with contiguous rank sets (DP over cut positions)
    best = [0] + [10 ** 9] * len(ranks)
    for j in range(len(ranks)):
        if best[j] >= 10 ** 9:
            continue
        lo = hi = ranks[j]
        for i in range(j, len(ranks)):
            lo, hi = min(lo, ranks[i]), max(hi, ranks[i])
            if hi - lo == i - j:
                best[i + 1] = min(best[i + 1], best[j] + 1)
    assert best[-1] <= st["waves"]


def test_call_output_table_validation():
    """bcss_plan_set_call_outputs: only for stop-level plans, one pointer per
    stop-level call (the fused S5 exchange's destination table)."""
    m, n, p, ba, bc = 4, 64, 64, 16, 16
    plain = bs.SttsmPlan(m, n, p, ba, bc)
    with pytest.raises(bs.NativeError):
        plain.set_call_outputs([0x1000])
    owner = bs.SttsmPlan(m, n, p, ba, bc, units=[1, 3], stop_level=m - 2)
    calls = owner.level_calls(m - 2)
    assert calls and all(c[-1] in (1, 3) for c in calls)
    with pytest.raises(bs.ShapeError):
        owner.set_call_outputs([0x1000] * (len(calls) + 1))
    owner.set_call_outputs([0x1000 + 8 * i for i in range(len(calls))])
    owner.set_call_outputs([])  # clears the table
