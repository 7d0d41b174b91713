"""BcssTensor / PartialSymTensor of the drop-in against the reference's
semantics (storage.py:44-170, tests/test_storage.py)."""

import itertools

import numpy as np
import pytest

import paper_1301_7744_b200 as bs
from conftest import GOLDEN
from oracle import bcss_oracle as orc


def _sym(m, n, seed):
    a = np.random.default_rng(seed).uniform(-1, 1, (n,) * m)
    return sum(np.transpose(a, p) for p in itertools.permutations(range(m))) / np.math.factorial(m) \
        if hasattr(np, "math") else None


def _symmetric(m, n, seed):
    import math
    a = np.random.default_rng(seed).uniform(-1, 1, (n,) * m)
    return sum(np.transpose(a, p) for p in itertools.permutations(range(m))) / math.factorial(m)


@pytest.mark.parametrize("m,nbar", [(2, 3), (3, 2), (3, 3), (4, 2)])
def test_block_at_matches_dense_subtensor(m, nbar):
    b = 2
    t = _symmetric(m, nbar * b, m + nbar)
    a = bs.BcssTensor(m, nbar * b, b, payload=orc.pack_dense(t, b))
    for idx in itertools.product(range(nbar), repeat=m):
        sl = tuple(slice(i * b, (i + 1) * b) for i in idx)
        assert np.allclose(a.block_at(idx), t[sl], atol=1e-15, rtol=0)
    assert np.allclose(a.to_dense(), t, atol=1e-15, rtol=0)


def test_payload_and_blocks_views_round_trip():
    d = np.load(GOLDEN / "sttsm_small_m4_n8_p8_ba4_bc4.npz")
    a = bs.BcssTensor(4, 8, 4, payload=d["A"])
    b = bs.BcssTensor(4, 8, 4, a.blocks)
    assert np.array_equal(b.payload, d["A"])
    assert a.dims == (8,) * 4 and a.grid == 2 and a.n == 8 and a.b == 4
    assert a.stored_element_count()[0] == 4**4 * bs.simplex_count(2, 4)


def test_matrix_redirect_hand_enumerated():
    # reference tests/test_storage.py:35-47: (1,0) -> stored (0,1) transposed
    t = _symmetric(2, 4, 3)
    a = bs.BcssTensor(2, 4, 2, payload=orc.pack_dense(t, 2))
    stored, axes = a.stored_and_transform((1, 0))
    assert axes == (1, 0)
    assert np.array_equal(stored, a.blocks[(0, 1)])
    assert np.array_equal(a.block_at((1, 0)), a.blocks[(0, 1)].T)


def test_validation():
    with pytest.raises(bs.BlockDivisibilityError):
        bs.BcssTensor(3, 6, 4, payload=np.zeros(1))
    with pytest.raises(bs.ShapeError):
        bs.BcssTensor(2, 4, 2, payload=np.zeros(5))
    with pytest.raises(bs.ShapeError):
        bs.BcssTensor(2, 4, 2, {(1, 0): np.zeros((2, 2)), (0, 0): np.zeros((2, 2)), (1, 1): np.zeros((2, 2))})
    a = bs.BcssTensor(2, 4, 2, payload=np.zeros(12))
    with pytest.raises(bs.RangeError):
        a.block_at((0, 2))


def test_reference_style_bcss_object_is_accepted_by_packing():
    class RefLike:  # duck-typed like blocksym.BcssTensor
        def __init__(self, a):
            self.order, self.n, self.b, self.blocks, self.tail_dims = 3, a.n, a.b, a.blocks, ()
    d = np.load(GOLDEN / "sttsm_config1.npz")
    a = bs.BcssTensor(3, 16, 4, payload=d["A"])
    assert np.array_equal(bs.packed_payload(RefLike(a)), d["A"])
