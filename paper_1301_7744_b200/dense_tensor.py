"""Dense tensors of the drop-in's host API.

``DenseTensor`` keeps the reference's contract
(/root/reference/pkg/src/blocksym/dense.py:78-116): an order-m array of
doubles in dimensional (Fortran) order exposed as ``.array``, with ``order``,
``dims``, ``data``, ``from_flat`` and ``copy``.  Block accessors of
``BcssTensor`` / ``PartialSymTensor`` and ``decompress`` return it, so code
written against the reference (``decompress(sttsm_bcss(...)).array``,
``a.block_at(idx).array``) runs unchanged.  It is host-side bookkeeping; the
arithmetic of the hot path never sees it.

``symmetry_violation`` restates the reference's check
(/root/reference/pkg/src/blocksym/indexing.py:71-107) that ``compress`` uses
to reject asymmetric input.
"""

from __future__ import annotations

import math
from typing import Iterable, Sequence

import numpy as np

from .errors import ShapeError


class DenseTensor:
    """Order-m array of doubles stored contiguously in dimensional order."""

    __slots__ = ("array",)

    def __init__(self, array):
        self.array = np.asfortranarray(array, dtype=np.float64)

    @classmethod
    def from_flat(cls, data, dims: Sequence[int]) -> "DenseTensor":
        """Build from a flat dimensional-order buffer and a dims tuple."""
        flat = np.asarray(data, dtype=np.float64)
        if flat.size != math.prod(dims):
            raise ShapeError(f"data length {flat.size} != product of dims {tuple(dims)}")
        return cls(flat.reshape(tuple(dims), order="F"))

    @property
    def order(self) -> int:
        return self.array.ndim

    @property
    def dims(self) -> tuple[int, ...]:
        return self.array.shape

    @property
    def data(self) -> np.ndarray:
        """Flat view of the buffer in dimensional order."""
        return self.array.reshape(-1, order="F")

    def copy(self) -> "DenseTensor":
        return DenseTensor(self.array.copy(order="F"))

    def __getitem__(self, idx):
        return self.array[idx]

    def __array__(self, dtype=None, copy=None):
        # lets numpy consumers (np.allclose, np.asarray) read it like an array
        arr = self.array if dtype is None else self.array.astype(dtype, copy=False)
        return arr.copy() if copy else arr

    def __repr__(self) -> str:
        return f"DenseTensor(dims={self.dims})"


def as_array(t) -> np.ndarray:
    """``t.array`` of a DenseTensor-like object (ours or the reference's), or
    ``t`` itself as an array."""
    arr = getattr(t, "array", t)
    return np.asarray(arr, dtype=np.float64)


def symmetry_violation(t, modes: Iterable[int]):
    """(max_rel, idx, swapped_idx): the worst relative mismatch
    |x - y| / max(|x|, |y|) of ``t`` under the adjacent transpositions of the
    sorted mode set (they generate every permutation of the set), with the
    index pair realizing it.  Same result as the reference's check
    (indexing.py:71-107)."""
    arr = as_array(t)
    group = sorted(set(modes))
    if any(not 0 <= s < arr.ndim for s in group):
        bad = next(s for s in group if not 0 <= s < arr.ndim)
        raise ShapeError(f"mode {bad} out of range for order {arr.ndim}")
    if len({arr.shape[s] for s in group}) > 1:
        raise ShapeError(f"modes {group} have unequal dimensions "
                         f"{sorted({arr.shape[s] for s in group})}")
    best_val, best_idx, best_jdx = 0.0, (0,) * arr.ndim, (0,) * arr.ndim
    for a, b in zip(group, group[1:]):
        other = np.swapaxes(arr, a, b)
        gap = np.abs(arr - other)
        rel = np.zeros(gap.shape)
        # gap > 0 implies max(|x|, |y|) > 0
        np.divide(gap, np.maximum(np.abs(arr), np.abs(other)), out=rel, where=gap > 0)
        pos = int(np.argmax(rel))
        val = float(rel.flat[pos])
        if val > best_val:
            idx = [int(i) for i in np.unravel_index(pos, rel.shape)]
            best_val, best_idx = val, tuple(idx)
            idx[a], idx[b] = idx[b], idx[a]
            best_jdx = tuple(idx)
    return best_val, best_idx, best_jdx
