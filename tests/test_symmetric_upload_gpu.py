"""Symmetric-aware upload of pipelined host runs (csrc/sym_upload.cu).

A BCSS tensor represents a symmetric tensor, so a block whose key repeats an
index holds every orbit of its repeated modes' permutations once
(storage.py:177-216: compress(t, b, tol=0) stores exactly symmetric blocks).
The symmetric upload moves only the sectors holding orbit representatives of
those blocks (zero-copy kernel) plus the distinct-key blocks (DMA), fills the
rest in HBM, and must give:
  * bit-identical C to the full upload when the blocks are exactly symmetric,
  * the oracle's C within 1e-12 relative Frobenius when they are symmetric
    only to rounding (the reference's random_bcss),
  * correct C across consecutive streamed calls (cumulative chunk counters and
    tickets, alternating device buffer sets),
and fall back to the full upload where it does not apply."""

import numpy as np
import pytest

import paper_1301_7744_b200 as bs
from oracle import bcss_oracle as orc
from paper_1301_7744_b200.dense import symmetrize_bcss_device

pytestmark = pytest.mark.gpu

CASES = [
    (3, 16, 16, 4, 4), (2, 64, 32, 8, 4), (3, 128, 96, 32, 16), (4, 64, 64, 16, 16),
    (4, 48, 32, 8, 8), (5, 32, 32, 8, 8), (6, 16, 16, 4, 4), (3, 256, 128, 64, 32),
    (4, 128, 64, 32, 32), (3, 96, 64, 32, 8),
]


def _pinned(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory()


def _exact_symmetric(m, n, b, seed):
    """random_bcss-style payload made exactly symmetric on the device
    (bcss_symmetrize_blocks: one value per orbit)."""
    import torch

    a = torch.from_numpy(orc.random_bcss_packed(m, n, b, seed)).cuda()
    symmetrize_bcss_device(a, m, n, b)
    torch.cuda.synchronize()
    return a.cpu().numpy()


def _host_run(plan, a, x):
    import torch

    c = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64).pin_memory()
    plan.run_host(_pinned(a).numpy(), _pinned(x).numpy(), c.numpy())
    return c.numpy().copy()


@pytest.mark.parametrize("cfg", CASES, ids=lambda c: "m%d_n%d_p%d_ba%d_bc%d" % c)
def test_symmetric_upload_bitwise_on_exact_symmetry(cfg):
    m, n, p, ba, bc = cfg
    rng = np.random.default_rng(sum(cfg) + 7)
    a = _exact_symmetric(m, n, ba, int(rng.integers(1 << 30)))
    x = rng.standard_normal((p, n))
    full = bs.SttsmPlan(m, n, p, ba, bc, pipeline=2)
    sym = bs.SttsmPlan(m, n, p, ba, bc, pipeline=2, symmetric_upload=True)
    c_full = _host_run(full, a, x)
    c_sym = _host_run(sym, a, x)
    assert full.last_upload_bytes == full.a_elems * 8
    assert sym.last_upload_bytes == sym.upload_bytes < sym.a_elems * 8
    assert np.array_equal(c_sym, c_full)
    assert orc.rel_frobenius(c_sym, orc.sttsm_bcss_packed(a, x, m, n, ba, bc)) <= 1e-12
    full.close()
    sym.close()


@pytest.mark.parametrize("cfg", CASES[:6], ids=lambda c: "m%d_n%d_p%d_ba%d_bc%d" % c)
def test_symmetric_upload_rounding_symmetric_input(cfg):
    # the reference's random_bcss averages over permutations: symmetric to ~1 ulp
    m, n, p, ba, bc = cfg
    rng = np.random.default_rng(sum(cfg) + 11)
    a = orc.random_bcss_packed(m, n, ba, int(rng.integers(1 << 30)))
    x = rng.standard_normal((p, n))
    plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=3, symmetric_upload=True)
    c = _host_run(plan, a, x)
    assert orc.rel_frobenius(c, orc.sttsm_bcss_packed(a, x, m, n, ba, bc)) <= 1e-12
    plan.close()


def test_symmetric_upload_streamed_calls():
    # consecutive streamed calls: alternating buffer sets, cumulative counters
    import torch

    m, n, p, ba, bc = 4, 64, 48, 16, 8
    plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=2, symmetric_upload=True)
    ins, outs, want = [], [], []
    for i in range(5):
        a = _exact_symmetric(m, n, ba, 100 + i)
        x = np.random.default_rng(200 + i).standard_normal((p, n))
        ins.append((_pinned(a), _pinned(x)))
        outs.append(torch.full((plan.c_elems,), float("nan"), dtype=torch.float64).pin_memory())
        want.append(orc.sttsm_bcss_packed(a, x, m, n, ba, bc))
    for rep in range(3):  # several rounds through the same plan
        for (ta, tx), tc in zip(ins, outs):
            tc.fill_(float("nan"))
            plan.run_host_async(ta.numpy(), tx.numpy(), tc.numpy())
        plan.wait()
        for tc, w in zip(outs, want):
            assert orc.rel_frobenius(tc.numpy(), w) <= 1e-12
    # and synchronous calls after the streamed ones
    for (ta, tx), w in zip(ins[:2], want[:2]):
        c = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64).pin_memory()
        plan.run_host(ta.numpy(), tx.numpy(), c.numpy())
        assert orc.rel_frobenius(c.numpy(), w) <= 1e-12
    plan.close()


def test_symmetric_upload_falls_back_where_it_does_not_apply():
    m, n, p, ba, bc = 3, 24, 12, 3, 2  # b_a = 3: not a power of two -> full upload
    rng = np.random.default_rng(5)
    a = orc.random_bcss_packed(m, n, ba, 9)
    x = rng.standard_normal((p, n))
    plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=2, symmetric_upload=True)
    assert plan.upload_bytes == plan.a_elems * 8
    c = _host_run(plan, a, x)
    assert plan.last_upload_bytes == plan.a_elems * 8
    assert orc.rel_frobenius(c, orc.sttsm_bcss_packed(a, x, m, n, ba, bc)) <= 1e-12
    # pageable A: staged through the plan's pinned buffers, then uploaded symmetrically
    plan2 = bs.SttsmPlan(3, 64, 32, 16, 16, pipeline=2, symmetric_upload=True)
    a2 = _exact_symmetric(3, 64, 16, 3)
    x2 = rng.standard_normal((32, 64))
    c2 = np.full(plan2.c_elems, np.nan)
    plan2.run_host(a2, x2, c2)
    assert orc.rel_frobenius(c2, orc.sttsm_bcss_packed(a2, x2, 3, 64, 16, 16)) <= 1e-12
    plan.close()
    plan2.close()


@pytest.mark.parametrize("env", [{"BCSS_SYM_GREEN": "1"}, {"BCSS_SYM_DMA": "0"}], ids=["green", "zc_all"])
def test_symmetric_upload_optional_modes(env, monkeypatch):
    # the SM partition (green contexts: upload kernel and compute on disjoint
    # SMs, streamed calls keep concurrent launches) and the all-zero-copy list:
    # same C bit for bit as the full upload, streamed and synchronous
    import torch

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    m, n, p, ba, bc = 4, 64, 48, 16, 8
    full = bs.SttsmPlan(m, n, p, ba, bc, pipeline=2)
    sym = bs.SttsmPlan(m, n, p, ba, bc, pipeline=2, symmetric_upload=True)
    ins = []
    for i in range(3):
        a = _exact_symmetric(m, n, ba, 300 + i)
        x = np.random.default_rng(400 + i).standard_normal((p, n))
        ins.append((_pinned(a), _pinned(x), _host_run(full, a, x)))
    outs = [torch.full((sym.c_elems,), float("nan"), dtype=torch.float64).pin_memory() for _ in ins]
    for rep in range(2):
        for (ta, tx, _), tc in zip(ins, outs):
            sym.run_host_async(ta.numpy(), tx.numpy(), tc.numpy())
        sym.wait()
        for (_, _, want), tc in zip(ins, outs):
            assert np.array_equal(tc.numpy(), want)
    ta, tx, want = ins[0]
    c = torch.full((sym.c_elems,), float("nan"), dtype=torch.float64).pin_memory()
    sym.run_host(ta.numpy(), tx.numpy(), c.numpy())
    assert np.array_equal(c.numpy(), want)
    assert sym.last_upload_bytes < 8 * sym.a_elems
    full.close()
    sym.close()


def test_dropin_symmetric_upload_on_compressed_tensor():
    # the reference idiom decompress(sttsm_bcss(compress(a, b), x, b_c)) with the
    # opt-in: compress(tol=0) guarantees exact symmetry, so C is bit-identical
    rng = np.random.default_rng(77)
    n, b, p, bc = 32, 8, 24, 8
    t = rng.uniform(-1, 1, (n, n, n))
    import itertools

    t = sum(np.transpose(t, perm) for perm in itertools.permutations(range(3))) / 6.0
    # exact symmetry: copy the canonical value into every permutation
    for i, j, k in itertools.product(range(n), repeat=3):
        s = tuple(sorted((i, j, k)))
        t[i, j, k] = t[s]
    a = bs.compress(t, b)
    x = rng.standard_normal((p, n))
    c_full = bs.sttsm_bcss(a, x, bc)
    c_sym = bs.sttsm_bcss(a, x, bc, symmetric_upload=True)
    assert np.array_equal(c_sym.payload, c_full.payload)
    assert np.array_equal(bs.decompress(c_sym).array, bs.decompress(c_full).array)
