"""CPU oracle for the BCSS ``sttsm`` hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain numpy restatement of the reference algorithm
(``blocksym.sttsm_bcss``, /root/reference/pkg/src/blocksym/change_of_basis.py:185-284)
and of the combinatorics it relies on.  It is the *checker*: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` leg may import it.  The product path (``paper_1301_7744_b200``)
never imports anything from ``oracle/`` and fails loudly when its CUDA library
is missing.

Parity is pinned: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by importing the reference package itself
(``oracle/gen_golden.py`` → ``tests/golden/*.npz``).

Data layout (same as the product's C-ABI): a BCSS tensor of order
``m``, dimension ``n`` and block dimension ``b`` is the *packed payload* — the
canonical blocks in ``hypertriangle_iter`` order, each ``b**m`` doubles in
dimensional (Fortran) order — exactly the ``.bcss`` file payload
(/root/reference/pkg/src/blocksym/io.py:50-55).  ``X`` is ``p x n`` row-major.
"""

from __future__ import annotations

import itertools
import math
from fractions import Fraction

import numpy as np

# --------------------------------------------------------------- combinatorics


def hypertriangle(extent: int, m: int) -> list[tuple[int, ...]]:
    """Nondecreasing m-tuples over 0..extent-1 in lex order.

    Restates ``hypertriangle_iter`` (indexing.py:57-61).
    """
    if extent < 1 or m < 1:
        raise ValueError("hypertriangle requires extent >= 1 and m >= 1")
    return list(itertools.combinations_with_replacement(range(extent), m))


def simplex_count(extent: int, m: int) -> int:
    """C(extent+m-1, m) (indexing.py:64-68)."""
    return math.comb(extent + m - 1, m)


def hypertriangle_rank(idx, extent: int) -> int:
    """Lex rank of a nondecreasing tuple among ``hypertriangle(extent, len(idx))``.

    Closed form: count the tuples that precede ``idx`` position by position
    (for each position t, all values v in [idx[t-1], idx[t]) give
    C(extent - v + (m-1-t) - 1, m-1-t) completions).
    """
    m = len(idx)
    r = 0
    lo = 0
    for t, v_hi in enumerate(idx):
        rem = m - 1 - t
        for v in range(lo, v_hi):
            r += math.comb(extent - v + rem - 1, rem) if rem > 0 else 1
        lo = v_hi
    return r


def canonical_mapping(idx) -> tuple[tuple[int, ...], tuple[int, ...]]:
    """(sorted idx, lexicographically smallest mapping) as in ``canonicalize``
    (indexing.py:34-54): first unused position of each value, in index order."""
    idx = tuple(idx)
    canonical = tuple(sorted(idx))
    next_pos: dict[int, int] = {}
    mapping = []
    for value in idx:
        pos = canonical.index(value, next_pos.get(value, 0))
        mapping.append(pos)
        next_pos[value] = pos + 1
    return canonical, tuple(mapping)


def insertion_position(key, ib: int) -> int:
    """Stored mode that holds logical mode ``k`` of the index ``key + (ib,)``.

    For sorted ``key`` the canonicalize mapping of ``key + (ib,)`` is the
    insertion permutation; ``ib`` lands at ``#{key entries <= ib}``
    (bisect-right), SURVEY §8(a) row a4.
    """
    return sum(1 for v in key if v <= ib)


# --------------------------------------------------------------- cost model


def bcss_flops(m: int, n: int, p: int, b_a: int, b_c: int, reuse: bool = True) -> int:
    """Exact blocked flop count (costs.py:83-112), in rational arithmetic."""
    nbar, pbar = n // b_a, p // b_c
    ratio = Fraction(b_c, b_a)

    def blocks_of(d):
        if not reuse:
            return nbar ** (m - 1 - d)
        return simplex_count(nbar, m - d - 1) if m - d - 1 >= 1 else 1

    core = sum(math.comb(pbar + d, d + 1) * blocks_of(d) * ratio**d for d in range(m))
    flops = 2 * nbar * b_c * b_a**m * core
    assert flops.denominator == 1
    return int(flops)


# --------------------------------------------------------------- inputs


def random_bcss_packed(m: int, n: int, b: int, seed: int) -> np.ndarray:
    """Seeded packed BCSS payload: U(-1,1) per canonical block, averaged over
    the modes of each repeated block index (restates generate.py:41-77, block
    by block, without materializing the dense tensor)."""
    rng = np.random.default_rng(seed)
    keys = hypertriangle(n // b, m)
    out = np.empty((len(keys), b**m), dtype=np.float64)
    for r, key in enumerate(keys):
        arr = rng.uniform(-1.0, 1.0, size=(b,) * m)
        groups: dict[int, list[int]] = {}
        for mode, kb in enumerate(key):
            groups.setdefault(kb, []).append(mode)
        for modes in groups.values():
            if len(modes) > 1:
                acc = np.zeros_like(arr)
                perms = list(itertools.permutations(modes))
                for perm in perms:
                    axes = list(range(m))
                    for src, dst in zip(modes, perm):
                        axes[src] = dst
                    acc += np.transpose(arr, axes)
                arr = acc / len(perms)
        out[r] = np.asfortranarray(arr).reshape(-1, order="F")
    return out.reshape(-1)


def pack_dense(t: np.ndarray, b: int) -> np.ndarray:
    """Canonical blocks of a dense symmetric tensor, packed (storage.py:177-217)."""
    m = t.ndim
    n = t.shape[0]
    keys = hypertriangle(n // b, m)
    out = np.empty((len(keys), b**m))
    for r, key in enumerate(keys):
        sl = tuple(slice(i * b, (i + 1) * b) for i in key)
        out[r] = t[sl].reshape(-1, order="F")
    return out.reshape(-1)


def unpack_dense(packed: np.ndarray, m: int, n: int, b: int) -> np.ndarray:
    """Dense tensor represented by a packed BCSS payload (storage.py:525-536)."""
    g = n // b
    blocks = packed.reshape(-1, b**m)
    out = np.empty((n,) * m, order="F")
    for idx in itertools.product(range(g), repeat=m):
        canonical, mapping = canonical_mapping(idx)
        blk = blocks[hypertriangle_rank(canonical, g)].reshape((b,) * m, order="F")
        sl = tuple(slice(i * b, (i + 1) * b) for i in idx)
        out[sl] = np.transpose(blk, mapping)
    return out


# --------------------------------------------------------------- algorithms


def sttsm_naive_dense(a: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Elementwise definition C[j] = sum_i A[i] prod_d X[j_d, i_d]
    (change_of_basis.py:77-110), as m successive tensordots."""
    c = a
    for _ in range(a.ndim):
        # contract the leading mode, append the new output mode at the end
        c = np.tensordot(c, x, axes=([0], [1]))
    return c


def pack_temp(blocks: dict, k: int, nbar: int) -> np.ndarray:
    """Packed payload of one temporary T(k) (canonical keys in hypertriangle order)."""
    return np.concatenate([blocks[key].reshape(-1, order="F") for key in hypertriangle(nbar, k)])


def sttsm_bcss_packed(a_packed: np.ndarray, x: np.ndarray, m: int, n: int, b_a: int,
                      b_c: int, keep_temps: bool = False, units=None, start=None):
    """Blocked change of basis over packed BCSS storage.

    Restates ``sttsm_bcss`` / ``_level_product`` (change_of_basis.py:185-284):
    depth-first walk over nondecreasing output block tuples; at level k each
    canonical key K of T(k) accumulates, over ib, X[jb rows, ib cols] times the
    stored block of T(k+1) at sorted(K ∪ {ib}) with its insertion position
    contracted.  Temporaries keep the reference block layout
    ``(b_a,)*k + (b_c,)*(m-k)`` (F-order).  Returns the packed C payload
    (blocks in hypertriangle order) and, with ``keep_temps``, a dict
    ``{(k, suffix): {key: block}}`` of every temporary.  ``units`` restricts
    the outermost loop to those jb_{m-1} values (a top-level subtree sample);
    C blocks outside them are left zero.  ``start=(L, {suffix: packed T(L)})``
    skips the levels above L and descends from the given temporaries only
    (the multi-GPU exchange point; ``a_packed`` is then unused).
    """
    x = np.asarray(x, dtype=np.float64)
    p = x.shape[0]
    nbar, pbar = n // b_a, p // b_c
    blk_a = b_a**m
    top = {}
    if start is None:
        a_blocks = a_packed.reshape(-1, blk_a)
        top = {key: a_blocks[r].reshape((b_a,) * m, order="F")
               for r, key in enumerate(hypertriangle(nbar, m))}
    c_keys = hypertriangle(pbar, m)
    c_out = np.zeros((len(c_keys), b_c**m))
    temps = {}

    def level(t_in: dict, k: int, jb: int) -> dict:
        rest = b_a**k * b_c ** (m - 1 - k)
        xr = x[jb * b_c:(jb + 1) * b_c]
        keys = hypertriangle(nbar, k) if k >= 1 else [()]
        produced = {}
        for key in keys:
            acc = np.zeros((b_c, rest))
            for ib in range(nbar):
                stored = t_in[tuple(sorted(key + (ib,)))]
                pos = insertion_position(key, ib)
                # front the contracted stored mode, keep the others in order
                axes = (pos,) + tuple(d for d in range(m) if d != pos)
                a_mat = np.transpose(stored, axes).reshape((b_a, rest), order="F")
                acc += xr[:, ib * b_a:(ib + 1) * b_a] @ a_mat
            fronted = acc.reshape((b_c,) + (b_a,) * k + (b_c,) * (m - 1 - k), order="F")
            inv = tuple(list(range(1, k + 1)) + [0] + list(range(k + 1, m)))
            produced[key] = np.asfortranarray(np.transpose(fronted, inv))
        return produced

    def descend(k: int, t_in: dict, j_hi: int, suffix: tuple) -> None:
        for jb in range(j_hi + 1):
            if k == m - 1 and units is not None and jb not in units:
                continue
            produced = level(t_in, k, jb)
            if k == 0:
                c_out[hypertriangle_rank((jb,) + suffix, pbar)] = \
                    produced[()].reshape(-1, order="F")
                continue
            if keep_temps:
                temps[(k, (jb,) + suffix)] = produced
            descend(k - 1, produced, jb, (jb,) + suffix)

    if start is None:
        descend(m - 1, top, pbar - 1, ())
    else:
        lvl, given = start
        shape = (b_a,) * lvl + (b_c,) * (m - lvl)
        size = int(np.prod(shape))
        for suffix, flat in given.items():
            t_in = {key: np.asarray(flat[r * size:(r + 1) * size]).reshape(shape, order="F")
                    for r, key in enumerate(hypertriangle(nbar, lvl))}
            descend(lvl - 1, t_in, suffix[0], tuple(suffix))
    c_packed = c_out.reshape(-1)
    return (c_packed, temps) if keep_temps else c_packed


def rel_frobenius(got: np.ndarray, want: np.ndarray) -> float:
    """||got - want||_F / ||want||_F over packed payloads (SURVEY §8d parity)."""
    den = float(np.linalg.norm(want))
    num = float(np.linalg.norm(np.asarray(got) - np.asarray(want)))
    return num / den if den > 0 else num


def max_rel(got: np.ndarray, want: np.ndarray) -> float:
    """max |got - want| / max |want| (change_of_basis.py:298-305)."""
    scale = float(np.max(np.abs(want)))
    diff = float(np.max(np.abs(np.asarray(got) - np.asarray(want))))
    return diff / scale if scale > 0 else diff
