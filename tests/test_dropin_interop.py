"""The drop-in's host objects against the reference's own code.

What ``sttsm_bcss`` returns must be consumable by code written for the
reference: ``decompress(sttsm_bcss(compress(a, b), x, b, c))``
(/root/reference/pkg/demos/02_change_of_basis.py:33,
pkg/tests/test_change_of_basis.py:135,147,231), ``cli.compare_bcss_dense``
and ``save_bcss``.  The CPU tests here build the exact object the drop-in
returns (a ``BcssTensor`` over the packed C payload) from the reference's
golden outputs and hand it to the reference package itself, imported
read-only from /root/reference (skipped where it is absent, e.g. on the GPU
box); the GPU tests at the bottom run the idiom end to end through the
CUDA path.
"""

import itertools
import math
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1301_7744_b200 as bs
from conftest import GOLDEN
from oracle import bcss_oracle as orc
from paper_1301_7744_b200 import sttsm as st_mod

REF_SRC = Path("/root/reference/pkg/src")


@pytest.fixture(scope="module")
def blocksym():
    if not (REF_SRC / "blocksym").is_dir():
        pytest.skip("reference package not present (it is not shipped to the GPU box)")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import blocksym
    import blocksym.cli  # noqa: F401  (compare_bcss_dense)

    return blocksym


def _symmetric(m, n, seed):
    a = np.random.default_rng(seed).uniform(-1, 1, (n,) * m)
    return sum(np.transpose(a, p) for p in itertools.permutations(range(m))) / math.factorial(m)


def _exact_symmetric(m, n, seed):
    """Exactly symmetric tensor: every entry is u[sorted(index)]."""
    u = np.random.default_rng(seed).uniform(-1, 1, (n,) * m)
    idx = np.sort(np.indices((n,) * m).reshape(m, -1), axis=0)
    return np.asfortranarray(u[tuple(idx)].reshape((n,) * m))


def _golden(name="sttsm_small_m4_n8_p8_ba4_bc4.npz"):
    d = np.load(GOLDEN / name)
    return d, tuple(int(v) for v in d["dims"])


# ---------------------------------------------------------------- CPU: host objects


def test_reference_decompress_accepts_drop_in_result(blocksym, tmp_path):
    d, (m, n, p, ba, bc) = _golden()
    result = bs.BcssTensor(m, p, bc, payload=d["C"])  # what sttsm_bcss returns
    dense_ref = blocksym.decompress(result)
    want = orc.unpack_dense(d["C"], m, p, bc)
    assert np.array_equal(dense_ref.array, want)
    assert np.array_equal(bs.decompress(result).array, want)
    # the reference's verification helper and file writer
    err, _ = blocksym.cli.compare_bcss_dense(result, blocksym.DenseTensor(want))
    assert err == 0.0
    blocksym.save_bcss(result, tmp_path / "ref.bcss")
    bs.save_bcss(result, tmp_path / "ours.bcss")
    assert (tmp_path / "ref.bcss").read_bytes() == (tmp_path / "ours.bcss").read_bytes()
    back = blocksym.load_bcss(tmp_path / "ours.bcss")
    assert np.array_equal(blocksym.decompress(back).array, want)


def test_reference_fault_injection_localises_block_on_drop_in_result(blocksym):
    """cli.verify_case(corrupt_block=...) replaces a block of the result
    (cli.py:121-122) and compare_bcss_dense names it; the replaced entry is
    also what our payload (the next GPU call's input) holds."""
    d, (m, n, p, ba, bc) = _golden()
    result = bs.BcssTensor(m, p, bc, payload=d["C"].copy())
    key = (0, 1, 1, 1)
    result.blocks[key] = result.blocks[key] + 1.0
    err, worst = blocksym.cli.compare_bcss_dense(result, blocksym.DenseTensor(orc.unpack_dense(d["C"], m, p, bc)))
    assert worst == key and err > 0
    r = orc.hypertriangle_rank(key, p // bc)
    bsz = bc**m
    assert np.array_equal(result.payload[r * bsz:(r + 1) * bsz], d["C"][r * bsz:(r + 1) * bsz] + 1.0)


def test_compress_matches_reference_and_round_trips(blocksym):
    t = _exact_symmetric(3, 12, 5)
    ours = bs.compress(bs.DenseTensor(t), 4)
    ref = blocksym.compress(blocksym.DenseTensor(t), 4)
    assert sorted(ours.blocks) == sorted(ref.blocks)
    for key, blk in ref.blocks.items():
        assert np.array_equal(ours.blocks[key], blk)
    assert np.array_equal(bs.decompress(ours).array, t)
    assert np.array_equal(blocksym.decompress(ours).array, t)
    # our decompress / packing read the reference's object too
    assert np.array_equal(bs.decompress(ref).array, t)
    assert np.array_equal(bs.packed_payload(ref), ours.payload)
    # partial compress (temporaries): leading group of 2 modes, one tail mode
    tp = np.ascontiguousarray(np.stack([_exact_symmetric(2, 6, s) for s in range(3)], axis=-1))
    part = bs.compress_partial(bs.DenseTensor(tp), 2, 3)
    refp = blocksym.compress_partial(blocksym.DenseTensor(tp), 2, 3)
    for key, blk in refp.blocks.items():
        assert np.array_equal(part.blocks[key], blk)
    assert np.array_equal(bs.decompress_partial(part).array, tp)


def test_compress_errors_and_symmetry_violation_match_reference(blocksym):
    rng = np.random.default_rng(4)
    bad = rng.standard_normal((4, 4))
    with pytest.raises(bs.SymmetryError) as ours:
        bs.compress(bs.DenseTensor(bad), 2)
    with pytest.raises(blocksym.SymmetryError) as ref:
        blocksym.compress(blocksym.DenseTensor(bad), 2)
    assert str(ours.value) == str(ref.value)
    with pytest.raises(bs.BlockDivisibilityError):
        bs.compress(bs.DenseTensor(_exact_symmetric(2, 4, 3)), 3)
    arr = _exact_symmetric(2, 4, 5)
    arr[1, 0] += 1e-14
    bs.compress(bs.DenseTensor(arr), 2, tol=1e-10)
    for seed in range(4):
        t = rng.standard_normal((3, 3, 3)) + _symmetric(3, 3, seed)
        assert bs.symmetry_violation(t, range(3)) == blocksym.symmetry_violation(blocksym.DenseTensor(t), range(3))


def test_block_accessors_return_dense_tensors_like_reference(blocksym):
    t = _exact_symmetric(3, 6, 8)
    ours = bs.compress(t, 2)
    ref = blocksym.compress(blocksym.DenseTensor(t), 2)
    for idx in itertools.product(range(3), repeat=3):
        c1, c2 = bs.OpCounter(), blocksym.OpCounter()
        a, b = ours.block_at(idx, c1), ref.block_at(idx, c2)
        assert isinstance(a, bs.DenseTensor) and a.dims == b.dims
        assert np.array_equal(a.array, b.array)
        assert c1.memops == c2.memops
    # canonical blocks are the stored buffer, without a copy
    assert np.shares_memory(ours.block_at((0, 1, 1)).array, ours.payload)
    ref_meta, our_meta = ref.meta[(1, 0, 2)], ours.meta[(1, 0, 2)]
    assert our_meta.canonical == ref_meta.canonical
    assert our_meta.applied.mapping == ref_meta.applied.mapping
    assert len(ours.meta) == len(ref.meta)


def test_drop_in_builds_reference_class_result(blocksym):
    """Given the reference's BcssTensor, the drop-in returns that class: the
    result object is built by sttsm._foreign_result from the packed C."""
    d, (m, n, p, ba, bc) = _golden()
    res = st_mod._foreign_result(blocksym.BcssTensor, m, p, bc, d["C"])
    assert isinstance(res, blocksym.BcssTensor)
    assert np.array_equal(blocksym.decompress(res).array, orc.unpack_dense(d["C"], m, p, bc))


def test_temp_to_dense_returns_dense_tensor():
    part = bs.PartialSymTensor(2, 4, 2, (3,), payload=np.arange(3 * 4 * 3, dtype=np.float64))
    out = bs.temp_to_dense(part)
    assert isinstance(out, bs.DenseTensor) and out.dims == (4, 4, 3)


def test_payload_follows_block_edits():
    """editing blocks after a run must not leave a stale payload.
    In-place edits land in the payload; replaced entries are copied in."""
    d, (m, n, p, ba, bc) = _golden()
    a = bs.BcssTensor(m, n, ba, payload=d["A"].copy())
    a.blocks[(0, 0, 0, 0)][0, 0, 0, 0] = 123.0
    assert a.payload[0] == 123.0
    a.blocks[(0, 0, 0, 1)] = np.full((ba,) * m, 7.0)
    bsz = ba**m
    assert np.all(a.payload[bsz:2 * bsz] == 7.0)
    # a tensor built from a blocks dict
    b = bs.BcssTensor(m, n, ba, {k: v.copy() for k, v in a.blocks.items()})
    assert np.array_equal(b.payload, a.payload)
    b.blocks[(1, 1, 1, 1)][...] = -1.0
    r = orc.hypertriangle_rank((1, 1, 1, 1), n // ba)
    assert np.all(b.payload[r * bsz:(r + 1) * bsz] == -1.0)


def test_partial_plan_host_buffers_are_sized_by_io_elems():
    """run_host of a start/stop plan moves the plan's own
    input/output sizes, which bcss_plan_io_elems reports (checked on CPU)."""
    m, n, p, ba, bc = 4, 8, 8, 2, 2
    stop = bs.SttsmPlan(m, n, p, ba, bc, stop_level=2)
    calls = stop.level_calls(2)
    assert stop.a_elems == bs.simplex_count(4, 4) * 2**4
    assert stop.c_elems == len(calls) * bs.simplex_count(4, 2) * 2**4 == 1600
    start = bs.SttsmPlan(m, n, p, ba, bc, start_level=2, start_calls=calls[:3])
    assert start.a_elems == 3 * bs.simplex_count(4, 2) * 2**4
    assert start.c_elems == bs.simplex_count(4, 4) * 2**4


# ---------------------------------------------------------------- GPU: the idiom end to end


class _RefLikeBcss:
    """Duck type of the reference's BcssTensor(order, dim, block_dim, blocks)
    (storage.py:155-170), for the GPU box where the reference is absent."""

    def __init__(self, order, dim, block_dim, blocks):
        self.order, self.n, self.b, self.blocks = order, dim, block_dim, blocks
        self.sym_modes, self.sym_dim, self.block_dim, self.tail_dims = order, dim, block_dim, ()
        self.grid = dim // block_dim

    @property
    def dims(self):
        return (self.n,) * self.order

    def partial_block_at(self, idx, counter=None):
        canonical = tuple(sorted(idx))
        _, mapping = orc.canonical_mapping(idx)
        return bs.DenseTensor(np.transpose(self.blocks[canonical], mapping))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sttsm_config1.npz", "sttsm_small_m4_n8_p8_ba4_bc4.npz",
                                  "sttsm_small_m3_n16_p32_ba4_bc16.npz", "sttsm_small_m5_n8_p8_ba4_bc4.npz"])
def test_decompress_sttsm_compress_idiom(name):
    """demos/02_change_of_basis.py:33: decompress(sttsm_bcss(compress(a, b), x, b_c))."""
    d, (m, n, p, ba, bc) = _golden(name)
    dense_a = bs.DenseTensor(orc.unpack_dense(d["A"], m, n, ba))
    # (the golden A's diagonal blocks carry ~1e-16 asymmetry from averaging,
    # so compress needs the tolerance the reference's tests use)
    c = bs.decompress(bs.sttsm_bcss(bs.compress(dense_a, ba, tol=1e-14), d["X"], bc))
    want = orc.unpack_dense(d["C"], m, p, bc)
    assert c.dims == (p,) * m
    assert orc.rel_frobenius(c.array, want) <= 1e-12
    naive = orc.sttsm_naive_dense(dense_a.array, d["X"])
    assert orc.max_rel(c.array, naive) <= 1e-10


@pytest.mark.gpu
def test_reference_shaped_object_in_gives_same_class_out():
    d, (m, n, p, ba, bc) = _golden()
    a_ref = _RefLikeBcss(m, n, ba, bs.BcssTensor(m, n, ba, payload=d["A"]).blocks)
    out = bs.sttsm_bcss(a_ref, d["X"], bc)
    assert isinstance(out, _RefLikeBcss)
    assert orc.rel_frobenius(bs.packed_payload(out), d["C"]) <= 1e-12
    assert orc.rel_frobenius(bs.decompress(out).array, orc.unpack_dense(d["C"], m, p, bc)) <= 1e-12


@pytest.mark.gpu
def test_repeated_calls_edit_between_runs():
    """Block edits between drop-in calls reach the GPU (no stale payload), and
    the registered payload / pooled pinned results stay correct across calls."""
    d, (m, n, p, ba, bc) = _golden("sttsm_small_m3_n64_p32_ba32_bc8.npz")
    a = bs.BcssTensor(m, n, ba, payload=d["A"].copy())
    first = bs.sttsm_bcss(a, d["X"], bc)
    assert orc.rel_frobenius(first.payload, d["C"]) <= 1e-12
    a.blocks[(0, 0, 0)][...] *= 2.0
    a.blocks[(1, 1, 1)] = a.blocks[(1, 1, 1)] * 3.0
    second = bs.sttsm_bcss(a, d["X"], bc)
    want = orc.sttsm_bcss_packed(a.payload.copy(), d["X"], m, n, ba, bc)
    assert orc.rel_frobenius(second.payload, want) <= 1e-12
    assert orc.rel_frobenius(first.payload, d["C"]) <= 1e-12  # first result untouched
    del first, second
    third = bs.sttsm_bcss(a, d["X"], bc)
    assert orc.rel_frobenius(third.payload, want) <= 1e-12


@pytest.mark.gpu
def test_run_host_on_partial_plans_matches_device_runs():
    """run_host of a stop-level plan returns T(stop) and a
    start plan consumes it, equal to the device runs of the same plans and,
    chained, to the reference C."""
    import torch

    d, (m, n, p, ba, bc) = _golden("sttsm_small_m4_n8_p8_ba4_bc4.npz")
    stop = bs.SttsmPlan(m, n, p, ba, bc, stop_level=2)
    t_host = np.full(stop.c_elems, np.nan)
    stop.run_host(np.ascontiguousarray(d["A"]), np.ascontiguousarray(d["X"]), t_host)
    t_dev = torch.full((stop.c_elems,), float("nan"), dtype=torch.float64, device="cuda")
    stop.run(torch.from_numpy(d["A"]).cuda(), torch.from_numpy(d["X"]).cuda(), t_dev)
    torch.cuda.synchronize()
    assert np.array_equal(t_host, t_dev.cpu().numpy())
    start = bs.SttsmPlan(m, n, p, ba, bc, start_level=2, start_calls=stop.level_calls(2))
    c_host = np.zeros(start.c_elems)
    start.run_host(t_host, np.ascontiguousarray(d["X"]), c_host)
    assert orc.rel_frobenius(c_host, d["C"]) <= 1e-12
    # a start plan over some calls writes only its own C blocks
    sub = bs.SttsmPlan(m, n, p, ba, bc, start_level=2, start_calls=stop.level_calls(2)[:1])
    c_sub = np.full(sub.c_elems, -7.0)
    blk = bs.simplex_count(n // ba, 2) * ba**2 * bc**2
    sub.run_host(np.ascontiguousarray(t_host[:blk]), np.ascontiguousarray(d["X"]), c_sub)
    ranks = sub.c_block_ranks()
    mask = np.zeros(bs.simplex_count(p // bc, m), bool)
    mask[ranks] = True
    bsz = bc**m
    got, want = c_sub.reshape(-1, bsz), np.asarray(d["C"]).reshape(-1, bsz)
    assert np.all(got[~mask] == -7.0)
    assert orc.rel_frobenius(got[mask], want[mask]) <= 1e-12


def _compare_bcss_dense(result, oracle_dense):
    """The reference's verification metric (cli.py:63-73): max relative error
    over stored blocks, and the worst block index."""
    scale = float(np.max(np.abs(oracle_dense))) or 1.0
    b = result.b
    worst = (0.0, next(iter(result.blocks)))
    for key, blk in result.blocks.items():
        sl = tuple(slice(i * b, (i + 1) * b) for i in key)
        err = float(np.max(np.abs(np.asarray(blk) - oracle_dense[sl]))) / scale
        if err > worst[0]:
            worst = (err, key)
    return worst


@pytest.mark.gpu
@pytest.mark.parametrize("key", [(0, 1, 2), (3, 3, 3), (0, 0, 3)])
def test_fault_injection_localises_corrupted_block(key):
    """cli.verify_case(corrupt_block=...) (cli.py:84,121-122;
    tests/test_cli.py:49-71): a block of the GPU result perturbed as the
    reference does it is the worst block against the naive oracle, and the
    unperturbed result passes the reference's 1e-10 bar."""
    d, (m, n, p, ba, bc) = _golden("sttsm_small_m3_n16_p16_ba4_bc2.npz")
    if max(key) >= p // bc:
        key = tuple(min(v, p // bc - 1) for v in key)
    out = bs.sttsm_bcss(bs.BcssTensor(m, n, ba, payload=d["A"]), d["X"], bc)
    naive = orc.sttsm_naive_dense(orc.unpack_dense(d["A"], m, n, ba), d["X"])
    err, _ = _compare_bcss_dense(out, naive)
    assert err <= 1e-10
    out.blocks[key] = out.blocks[key] + 1.0
    err, worst = _compare_bcss_dense(out, naive)
    assert worst == key and err > 1e-3
    # the corruption is what the next GPU call would read, too
    r = orc.hypertriangle_rank(key, p // bc)
    assert np.allclose(out.payload[r * bc**m:(r + 1) * bc**m], np.asarray(out.blocks[key]).reshape(-1, order="F"))
