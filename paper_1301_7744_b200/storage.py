"""BCSS tensor objects of the drop-in.

Same constructor, attributes and accessors as the reference's
``PartialSymTensor`` / ``BcssTensor`` and the same ``compress`` /
``decompress`` functions (/root/reference/pkg/src/blocksym/storage.py:44-236),
backed by the *packed payload* the GPU consumes: canonical blocks in
hypertriangle order, each in dimensional (Fortran) order (io.py:50-55).

* ``payload`` is the storage.  A tensor built from a ``blocks`` dict copies
  the blocks into a payload once (in pinned host memory when a GPU is
  present, so host runs move it by DMA without staging, ``hostmem.py``).
* ``blocks`` is a dict of F-order views into the payload, so the reference's
  idioms keep working: in-place edits ``t.blocks[key][...] = v`` land in the
  payload directly, and an entry replaced by a new array
  (``t.blocks[key] = arr``, as ``cli.verify_case(corrupt_block=...)`` does)
  is detected by identity and copied into its slot whenever the payload is
  read.  The dict stays the source of truth, as in the reference.
* Block accessors return ``DenseTensor`` (``.array``), canonical blocks
  without a copy, others as permuted copies counted as memops
  (storage.py:131-142, dense.py:133-147).

The reference keeps a dense meta-grid of ``grid**s`` redirection records
(storage.py:98-101); here ``meta`` is a lazy mapping that computes the same
record with ``canonicalize`` on lookup (the tie-break is the same,
indexing.py:45-54), because the device path never needs a host meta-grid.
"""

from __future__ import annotations

import itertools
import math
from collections.abc import Mapping
from typing import NamedTuple

import numpy as np

from .counters import OpCounter
from .dense_tensor import DenseTensor, as_array, symmetry_violation
from .errors import BlockDivisibilityError, RangeError, ShapeError, SymmetryError
from .hostmem import host_empty
from .indexing import MultiIndex, canonicalize, hypertriangle_iter, simplex_count


class AppliedPermutation(NamedTuple):
    """Mode mapping of a redirection record: position d of the logical block
    is mode ``mapping[d]`` of the stored block."""

    mapping: tuple[int, ...]

    def is_identity(self) -> bool:
        return all(j == d for d, j in enumerate(self.mapping))


class CanonicalRef(NamedTuple):
    """Redirection record of one block index (indexing.py CanonicalRef)."""

    canonical: MultiIndex
    applied: AppliedPermutation


class MetaGrid(Mapping):
    """The reference's meta-grid as a lazy mapping: every index of the
    ``grid**sym_modes`` block grid → its ``CanonicalRef``, computed on lookup."""

    def __init__(self, grid: int, sym_modes: int):
        self.grid, self.sym_modes = grid, sym_modes

    def __getitem__(self, idx) -> CanonicalRef:
        idx = tuple(idx)
        if len(idx) != self.sym_modes or any(not (isinstance(i, (int, np.integer)) and 0 <= i < self.grid)
                                             for i in idx):
            raise KeyError(idx)
        canonical, mapping = canonicalize(idx)
        return CanonicalRef(canonical, AppliedPermutation(mapping))

    def __iter__(self):
        return itertools.product(range(self.grid), repeat=self.sym_modes)

    def __len__(self) -> int:
        return self.grid ** self.sym_modes


class PartialSymTensor:
    """Blocked store for a tensor symmetric in its leading ``sym_modes`` modes.

    ``blocks`` maps nondecreasing ``sym_modes``-tuples to arrays of shape
    ``(block_dim,)*sym_modes + tail_dims``; alternatively pass ``payload``, the
    packed 1-D buffer (numpy, length ``simplex_count(grid, s) * block_size``),
    which the tensor then views without copying.
    """

    def __init__(self, sym_modes: int, sym_dim: int, block_dim: int,
                 tail_dims: tuple[int, ...], blocks: dict | None = None, *, payload=None):
        if sym_modes < 1:
            raise ShapeError("need at least one symmetric mode")
        if block_dim < 1 or sym_dim % block_dim != 0:
            raise BlockDivisibilityError(f"block dimension {block_dim} does not divide {sym_dim}")
        self.sym_modes = sym_modes
        self.sym_dim = sym_dim
        self.block_dim = block_dim
        self.tail_dims = tuple(tail_dims)
        self.grid = sym_dim // block_dim
        self.block_shape = (block_dim,) * sym_modes + self.tail_dims
        self.block_size = math.prod(self.block_shape)
        self.n_blocks = simplex_count(self.grid, sym_modes)
        self._blocks = None   # key -> array (views into the payload unless replaced)
        self._views = None    # key -> the payload view handed out for it
        if (blocks is None) == (payload is None):
            raise ShapeError("pass exactly one of blocks / payload")
        if blocks is not None:
            if len(blocks) != self.n_blocks:
                raise ShapeError(f"expected {self.n_blocks} canonical blocks, got {len(blocks)}")
            for key, arr in blocks.items():
                if tuple(sorted(key)) != tuple(key):
                    raise ShapeError(f"block key {key} is not nondecreasing")
                if np.shape(arr) != self.block_shape:
                    raise ShapeError(f"block {key} has shape {np.shape(arr)}, expected {self.block_shape}")
                if any(not 0 <= i < self.grid for i in key) or len(key) != sym_modes:
                    raise RangeError(f"block key {key} outside grid {self.grid}^{sym_modes}")
            self._payload = host_empty(self.n_blocks * self.block_size)
            bs = self.block_size
            for r, key in enumerate(hypertriangle_iter(self.grid, sym_modes)):
                self._payload[r * bs:(r + 1) * bs] = np.asarray(blocks[key], dtype=np.float64).reshape(
                    -1, order="F")
        else:
            flat = np.asarray(payload, dtype=np.float64).reshape(-1)
            if flat.size != self.n_blocks * self.block_size:
                raise ShapeError(f"payload of {flat.size} elements, expected "
                                 f"{self.n_blocks * self.block_size}")
            self._payload = flat

    # ---- views ------------------------------------------------------------------
    @property
    def payload(self) -> np.ndarray:
        """Packed canonical blocks (hypertriangle order, F-order blocks).
        ``blocks`` entries that were replaced by other arrays are copied into
        their slots first, so the payload always equals what ``blocks`` holds."""
        if self._blocks is not None:
            for key, view in self._views.items():
                cur = self._blocks[key]
                if cur is not view:
                    if np.shape(cur) != self.block_shape:
                        raise ShapeError(f"block {key} has shape {np.shape(cur)}, expected {self.block_shape}")
                    view[...] = cur
        return self._payload

    @property
    def blocks(self) -> dict:
        if self._blocks is None:
            flat = self._payload
            bs = self.block_size
            self._views = {
                key: flat[r * bs:(r + 1) * bs].reshape(self.block_shape, order="F")
                for r, key in enumerate(hypertriangle_iter(self.grid, self.sym_modes))
            }
            self._blocks = dict(self._views)
        return self._blocks

    @property
    def meta(self) -> MetaGrid:
        return MetaGrid(self.grid, self.sym_modes)

    @property
    def order(self) -> int:
        return self.sym_modes + len(self.tail_dims)

    @property
    def dims(self) -> tuple[int, ...]:
        return (self.sym_dim,) * self.sym_modes + self.tail_dims

    def __repr__(self) -> str:
        return f"{type(self).__name__}(dims={self.dims}, b={self.block_dim}, blocks={self.n_blocks})"

    # ---- redirection (storage.py:123-142) ---------------------------------------
    def stored_and_transform(self, sym_idx: MultiIndex):
        sym_idx = tuple(sym_idx)
        if len(sym_idx) != self.sym_modes or any(not 0 <= i < self.grid for i in sym_idx):
            raise RangeError(f"block index {sym_idx} outside grid {self.grid}^{self.sym_modes}")
        canonical, mapping = canonicalize(sym_idx)
        tail = tuple(range(self.sym_modes, self.order))
        return self.blocks[canonical], mapping + tail

    def partial_block_at(self, sym_idx: MultiIndex, counter: OpCounter | None = None) -> DenseTensor:
        """Logical block at ``sym_idx``: the stored block itself for a
        canonical index, else a copy with the recorded permutation applied to
        the symmetric modes (2 memops per element on ``counter``)."""
        stored, axes = self.stored_and_transform(sym_idx)
        if axes == tuple(range(len(axes))):
            return DenseTensor(stored)
        out = np.array(np.transpose(stored, axes), order="F", copy=True)
        if counter is not None:
            counter.count_memops(2 * out.size)
        return DenseTensor(out)

    def stored_element_count(self, meta_k: float = 0) -> tuple[int, float]:
        payload = self.n_blocks * self.block_size
        return payload, payload + meta_k * self.grid**self.sym_modes

    def to_dense(self) -> np.ndarray:
        """The dense tensor this store represents, as an F-order array."""
        return decompress_partial(self).array


class BcssTensor(PartialSymTensor):
    """Fully symmetric tensor stored by canonical blocks (storage.py:155-170)."""

    def __init__(self, order: int, dim: int, block_dim: int, blocks: dict | None = None, *,
                 payload=None):
        super().__init__(order, dim, block_dim, (), blocks, payload=payload)

    @property
    def n(self) -> int:
        return self.sym_dim

    @property
    def b(self) -> int:
        return self.block_dim

    def block_at(self, idx: MultiIndex, counter: OpCounter | None = None) -> DenseTensor:
        return self.partial_block_at(idx, counter)


def packed_payload(a) -> np.ndarray:
    """Packed payload of any BCSS-like object: ours, or the reference's
    ``BcssTensor`` (blocks dict keyed by sorted tuples), packed fresh into
    pinned memory (the packing copy doubles as the DMA staging)."""
    if isinstance(a, PartialSymTensor):
        return a.payload
    grid = a.n // a.b
    bs = a.b ** a.order
    out = host_empty(simplex_count(grid, a.order) * bs)
    for r, key in enumerate(hypertriangle_iter(grid, a.order)):
        out[r * bs:(r + 1) * bs] = np.asarray(a.blocks[key], dtype=np.float64).reshape(-1, order="F")
    return out


# ---- compress / decompress (storage.py:177-236) ---------------------------------

def compress_partial(t, sym_modes: int, block_dim: int, tol: float = 0.0) -> PartialSymTensor:
    """Store ``t`` (symmetric in modes ``0..sym_modes-1``) by canonical blocks,
    copied verbatim into a packed payload; raises ``SymmetryError`` naming the
    worst index pair when the symmetry does not hold within ``tol``."""
    arr = as_array(t)
    m = arr.ndim
    if not 0 < sym_modes <= m:
        raise ShapeError(f"sym_modes {sym_modes} not in 1..{m}")
    if len(set(arr.shape[:sym_modes])) > 1:
        raise ShapeError(f"symmetric modes have unequal dimensions {arr.shape[:sym_modes]}")
    n = arr.shape[0]
    if block_dim < 1 or n % block_dim != 0:
        raise BlockDivisibilityError(f"block dimension {block_dim} does not divide {n}")
    if sym_modes > 1:
        rel, idx, jdx = symmetry_violation(arr, range(sym_modes))
        if rel > tol:
            raise SymmetryError(f"asymmetry {rel:.3e} > tol {tol:.3e} between indices {idx} and {jdx}")
    grid = n // block_dim
    tail_dims = tuple(arr.shape[sym_modes:])
    bs = block_dim**sym_modes * math.prod(tail_dims)
    payload = host_empty(simplex_count(grid, sym_modes) * bs)
    tail = (slice(None),) * len(tail_dims)
    for r, key in enumerate(hypertriangle_iter(grid, sym_modes)):
        sl = tuple(slice(i * block_dim, (i + 1) * block_dim) for i in key) + tail
        payload[r * bs:(r + 1) * bs] = arr[sl].reshape(-1, order="F")
    return PartialSymTensor(sym_modes, n, block_dim, tail_dims, payload=payload)


def compress(t, block_dim: int, tol: float = 0.0) -> BcssTensor:
    """Store a fully symmetric tensor by canonical blocks."""
    arr = as_array(t)
    if len(set(arr.shape)) > 1:
        raise ShapeError(f"tensor dims {tuple(arr.shape)} are not all equal")
    part = compress_partial(arr, arr.ndim, block_dim, tol)
    return BcssTensor(arr.ndim, part.sym_dim, block_dim, payload=part.payload)


def decompress_partial(a, counter: OpCounter | None = None) -> DenseTensor:
    """Dense tensor a blocked store represents (ours or the reference's):
    every grid index filled from its logical block."""
    out = np.empty(a.dims, dtype=np.float64, order="F")
    b = a.block_dim
    tail = (slice(None),) * len(a.tail_dims)
    for key in itertools.product(range(a.grid), repeat=a.sym_modes):
        sl = tuple(slice(i * b, (i + 1) * b) for i in key) + tail
        out[sl] = a.partial_block_at(key, counter).array
    return DenseTensor(out)


def decompress(a, counter: OpCounter | None = None) -> DenseTensor:
    return decompress_partial(a, counter)
