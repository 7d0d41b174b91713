"""Block-index combinatorics used by the host layer.

Interfaces follow the reference (/root/reference/pkg/src/blocksym/indexing.py):
``hypertriangle_iter`` (:57-61), ``simplex_count`` (:64-68) and
``canonicalize`` (:34-54).  The rank / unrank functions are the packed-payload
slot of a canonical block; they are computed by the native library (the same
code the device tables are built from) so the host and device agree.
"""

from __future__ import annotations

import ctypes
import itertools
import math
from typing import Iterable, Iterator

from . import _native
from .errors import ParameterError

MultiIndex = tuple[int, ...]


def hypertriangle_iter(extent: int, m: int) -> Iterator[MultiIndex]:
    """Every nondecreasing m-tuple over ``0..extent-1`` in lex order."""
    if extent < 1 or m < 1:
        raise ParameterError("hypertriangle_iter requires extent >= 1 and m >= 1")
    return itertools.combinations_with_replacement(range(extent), m)


def simplex_count(n: int, m: int) -> int:
    """Number of nondecreasing m-tuples over ``0..n-1``: C(n + m - 1, m)."""
    if n < 1 or m < 1:
        raise ParameterError("simplex_count requires n >= 1 and m >= 1")
    return math.comb(n + m - 1, m)


def canonicalize(idx: Iterable[int]) -> tuple[MultiIndex, MultiIndex]:
    """(sorted index, lexicographically smallest mapping) with
    ``canonical[mapping[d]] == idx[d]``; ties resolved by first unused slot."""
    idx = tuple(idx)
    canonical = tuple(sorted(idx))
    next_pos: dict[int, int] = {}
    mapping = []
    for value in idx:
        pos = canonical.index(value, next_pos.get(value, 0))
        mapping.append(pos)
        next_pos[value] = pos + 1
    return canonical, tuple(mapping)


def hypertriangle_rank(idx: Iterable[int], extent: int) -> int:
    """Slot of the canonical block ``idx`` in a packed payload (native)."""
    idx = tuple(int(v) for v in idx)
    arr = (ctypes.c_int64 * len(idx))(*idx)
    out = ctypes.c_int64()
    _native.check(_native.lib().bcss_hypertriangle_rank(arr, len(idx), extent, ctypes.byref(out)))
    return int(out.value)


def hypertriangle_unrank(rank: int, m: int, extent: int) -> MultiIndex:
    arr = (ctypes.c_int64 * m)()
    _native.check(_native.lib().bcss_hypertriangle_unrank(rank, m, extent, arr))
    return tuple(int(v) for v in arr)
