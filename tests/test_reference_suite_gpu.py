"""The reference's own blocked-algorithm tests, re-run through the drop-in.

Mirrors the ``sttsm_bcss`` cases of the reference test suite
(/root/reference/pkg/tests/test_change_of_basis.py:113-231) case by case —
same shapes, same tolerances, same assertions — with the reference's helpers
restated here (dense symmetric input by averaging over all mode permutations,
compression to BCSS = ``oracle.pack_dense``) and the reference's naive
algorithm (change_of_basis.py:77-110) restated as one ``np.einsum`` over all
modes.  Every case runs
on the GPU through ``sttsm_bcss`` (C ABI -> sm_100a DMMA kernels).
"""

import itertools
import math

import numpy as np
import pytest

import paper_1301_7744_b200 as bs
from oracle import bcss_oracle as orc

pytestmark = pytest.mark.gpu

_LETTERS = "abcdefgh"


def random_symmetric(m: int, n: int, seed: int) -> np.ndarray:
    """Dense symmetric tensor: U(-1,1) averaged over all m! mode permutations."""
    t = np.random.default_rng(seed).uniform(-1.0, 1.0, (n,) * m)
    return sum(np.transpose(t, perm) for perm in itertools.permutations(range(m))) / math.factorial(m)


def random_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal((rows, cols))


def compress(a: np.ndarray, b: int) -> bs.BcssTensor:
    return bs.BcssTensor(a.ndim, a.shape[0], b, payload=orc.pack_dense(a, b))


def decompress(t: bs.BcssTensor) -> np.ndarray:
    return orc.unpack_dense(t.payload, t.order, t.n, t.b)


def sttsm_naive(a: np.ndarray, x: np.ndarray) -> np.ndarray:
    """C[j_0..j_{m-1}] = sum_i A[i_0..i_{m-1}] prod_d X[j_d, i_d], one einsum."""
    m = a.ndim
    ins, outs = _LETTERS[:m], _LETTERS[:m].upper()
    spec = ins + "," + ",".join(outs[d] + ins[d] for d in range(m)) + "->" + outs
    return np.einsum(spec, a, *([x] * m), optimize=True)


def max_relative_error(got: np.ndarray, want: np.ndarray) -> float:
    """The reference's metric (cli.py:63-73): max |got - want| / max |want|."""
    return float(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-300))


def is_sym_in_modes(t: np.ndarray, modes, tol: float) -> bool:
    modes = list(modes)
    scale = max(np.max(np.abs(t)), 1e-300)
    for i, j in zip(modes, modes[1:]):
        perm = list(range(t.ndim))
        perm[i], perm[j] = perm[j], perm[i]
        if np.max(np.abs(t - np.transpose(t, perm))) > tol * scale:
            return False
    return True


def exactly_symmetric(m: int, n: int, seed: int) -> np.ndarray:
    """A[i] = U[sorted(i)]: symmetric to the last bit (averaging over
    permutations leaves ~1e-16 asymmetry inside diagonal blocks, which a
    redirected read exposes)."""
    u = np.random.default_rng(seed).uniform(-1.0, 1.0, (n,) * m)
    idx = np.sort(np.indices((n,) * m).reshape(m, -1), axis=0)
    return u[tuple(idx)].reshape((n,) * m)


def test_bcss_identity_matrix_returns_input():
    # test_change_of_basis.py:33-36 (naive flavour), here for the blocked path:
    # X = I reproduces A exactly (every output is one product by 1.0 plus
    # zeros, read through the redirection permutations)
    packed = compress(exactly_symmetric(3, 8, 11), 4)
    out = bs.sttsm_bcss(packed, np.eye(8), 4)
    np.testing.assert_array_equal(out.payload, packed.payload)


def test_bcss_m2_sandwich():
    # test_change_of_basis.py:95-99: order 2 is X A X^T
    a = random_symmetric(2, 6, 12)
    x = random_matrix(6, 6, 13)
    out = bs.sttsm_bcss(compress(a, 3), x, 3)
    want = x @ a @ x.T
    assert max_relative_error(decompress(out), want) < 1e-13


def test_bcss_degenerate_single_block_equals_dense_chain():
    # test_change_of_basis.py:113-123
    a = random_symmetric(3, 4, 17)
    x = random_matrix(4, 4, 18)
    out = bs.sttsm_bcss(compress(a, 4), x, 4)
    assert len(out.blocks) == 1
    dense = orc.sttsm_naive_dense(a, x)
    scale = np.max(np.abs(dense))
    assert np.max(np.abs(out.blocks[(0, 0, 0)] - dense)) / scale < 1e-13


@pytest.mark.parametrize("m", [2, 3, 4])
@pytest.mark.parametrize("n", [4, 6])
@pytest.mark.parametrize("b", [1, 2])
def test_bcss_matches_naive_reduced_sweep(m, n, b):
    # test_change_of_basis.py:126-136
    a = random_symmetric(m, n, m * 31 + n)
    x = random_matrix(n, n, m * 37 + n)
    packed = compress(a, b)
    want = sttsm_naive(a, x)
    for reuse in (True, False):
        out = bs.sttsm_bcss(packed, x, b, reuse=reuse)
        got = decompress(out)
        err = max_relative_error(got, want)
        assert err < 1e-10, (m, n, b, reuse, err)
        assert orc.rel_frobenius(got, want) <= 1e-12


def test_bcss_rectangular_blocks_and_output_dim():
    # test_change_of_basis.py:139-148: p != n and b_C != b_A
    a = random_symmetric(3, 6, 19)
    x = random_matrix(4, 6, 20)
    out = bs.sttsm_bcss(compress(a, 3), x, 2)
    assert out.dims == (4, 4, 4)
    assert len(out.blocks) == bs.simplex_count(2, 3)
    assert max_relative_error(decompress(out), sttsm_naive(a, x)) < 1e-10


def test_bcss_output_block_count():
    # test_change_of_basis.py:151-156
    a = random_symmetric(4, 4, 21)
    x = random_matrix(4, 4, 22)
    out = bs.sttsm_bcss(compress(a, 2), x, 1)
    assert len(out.blocks) == bs.simplex_count(4, 4)


@pytest.mark.parametrize("m,n,b", [(2, 4, 1), (2, 4, 2), (3, 4, 2), (3, 8, 4), (2, 8, 2)])
def test_bcss_counter_equals_formula_both_modes(m, n, b):
    # test_change_of_basis.py:159-169: the counter gets the cost model's flops
    a = random_symmetric(m, n, m + n + b)
    x = random_matrix(n, n, m + n + b + 1)
    packed = compress(a, b)
    for reuse in (True, False):
        c = bs.OpCounter()
        bs.sttsm_bcss(packed, x, b, c, reuse=reuse)
        assert c.flops == orc.bcss_flops(m, n, n, b, b, reuse=reuse), (m, n, b, reuse)
        assert c.memops == bs.bcss_memops(m, n, n, b, b, reuse=reuse)


def test_bcss_temporaries_are_partially_symmetric():
    # test_change_of_basis.py:172-188
    a = random_symmetric(4, 4, 23)
    x = random_matrix(4, 4, 24)
    audited = []

    def hook(k, temp):
        dense = bs.temp_to_dense(temp)  # a DenseTensor, as in the reference
        audited.append((k, dense.dims))
        assert is_sym_in_modes(dense.array, range(k), 1e-12), k

    bs.sttsm_bcss(compress(a, 2), x, 2, temp_hook=hook)
    assert {k for k, _ in audited} == {1, 2, 3}
    for k, dims in audited:
        assert dims == (4,) * k + (2,) * (4 - k)


def test_bcss_temp_hook_no_reuse_flavor():
    # test_change_of_basis.py:191-198
    a = random_symmetric(3, 4, 25)
    x = random_matrix(4, 4, 26)
    seen = []
    bs.sttsm_bcss(compress(a, 2), x, 2, reuse=False, temp_hook=lambda k, t: seen.append((k, bs.temp_to_dense(t))))
    assert seen
    for k, dense in seen:
        assert bs.symmetry_violation(dense, range(k))[0] <= 1e-12 if k >= 2 else True


def test_bcss_validations():
    # test_change_of_basis.py:201-207
    packed = compress(random_symmetric(3, 4, 27), 2)
    with pytest.raises(bs.BlockDivisibilityError):
        bs.sttsm_bcss(packed, random_matrix(4, 4, 28), 3)
    with pytest.raises(bs.ShapeError):
        bs.sttsm_bcss(packed, random_matrix(4, 5, 29), 2)


@pytest.mark.parametrize("m", [2, 3, 4, 5])
@pytest.mark.parametrize("n", [4, 6, 8])
def test_all_algorithms_agree(m, n):
    # test_change_of_basis.py:220-231: blocked (every block size dividing n
    # that the reference sweeps) and the dense GPU chain against the naive sum
    import torch

    from paper_1301_7744_b200 import dense

    a = random_symmetric(m, n, m * 41 + n)
    x = random_matrix(n, n, m * 43 + n)
    oracle = sttsm_naive(a, x)
    ttm = dense.sttsm_dense_ttm_device(torch.from_numpy(a).cuda(), torch.from_numpy(x).cuda()).cpu().numpy()
    assert max_relative_error(ttm, oracle) < 1e-10
    for b in sorted({1, 2, n // 2, n}):
        out = bs.sttsm_bcss(compress(a, b), x, b)
        assert max_relative_error(decompress(out), oracle) < 1e-10, (m, n, b)
