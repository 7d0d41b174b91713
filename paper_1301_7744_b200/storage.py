"""BCSS tensor objects of the drop-in.

Same constructor and attributes as the reference's ``PartialSymTensor`` /
``BcssTensor`` (/root/reference/pkg/src/blocksym/storage.py:44-170), backed by
the *packed payload* the GPU consumes: canonical blocks in hypertriangle
order, each in dimensional (Fortran) order (io.py:50-55).  Either view is
built lazily from the other, so a device result is wrapped without copying
block by block, and a reference-built ``blocks`` dict packs once.

The reference keeps a dense meta-grid of ``grid**s`` redirection records
(storage.py:98-101); here redirection is computed on demand with
``canonicalize`` (the tie-break is the same, indexing.py:45-54), because the
device path never needs a host meta-grid.
"""

from __future__ import annotations

import itertools
import math

import numpy as np

from .errors import BlockDivisibilityError, RangeError, ShapeError
from .indexing import MultiIndex, canonicalize, hypertriangle_iter, simplex_count


class PartialSymTensor:
    """Blocked store for a tensor symmetric in its leading ``sym_modes`` modes.

    ``blocks`` maps nondecreasing ``sym_modes``-tuples to arrays of shape
    ``(block_dim,)*sym_modes + tail_dims``; alternatively pass ``payload``, the
    packed 1-D buffer (numpy, length ``simplex_count(grid, s) * block_size``).
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
        self._blocks = None
        self._payload = None
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
            self._blocks = dict(blocks)
        else:
            flat = np.asarray(payload, dtype=np.float64).reshape(-1)
            if flat.size != self.n_blocks * self.block_size:
                raise ShapeError(f"payload of {flat.size} elements, expected "
                                 f"{self.n_blocks * self.block_size}")
            self._payload = flat

    # ---- views ------------------------------------------------------------------
    @property
    def payload(self) -> np.ndarray:
        """Packed canonical blocks (hypertriangle order, F-order blocks)."""
        if self._payload is None:
            out = np.empty(self.n_blocks * self.block_size, dtype=np.float64)
            for r, key in enumerate(hypertriangle_iter(self.grid, self.sym_modes)):
                out[r * self.block_size:(r + 1) * self.block_size] = \
                    np.asarray(self._blocks[key], dtype=np.float64).reshape(-1, order="F")
            self._payload = out
        return self._payload

    @property
    def blocks(self) -> dict:
        if self._blocks is None:
            flat = self._payload
            bs = self.block_size
            self._blocks = {
                key: flat[r * bs:(r + 1) * bs].reshape(self.block_shape, order="F")
                for r, key in enumerate(hypertriangle_iter(self.grid, self.sym_modes))
            }
        return self._blocks

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

    def partial_block_at(self, sym_idx: MultiIndex) -> np.ndarray:
        """Logical block at ``sym_idx`` (stored block with the recorded
        permutation applied to the symmetric modes)."""
        stored, axes = self.stored_and_transform(sym_idx)
        if axes == tuple(range(len(axes))):
            return stored
        return np.asfortranarray(np.transpose(stored, axes))

    def stored_element_count(self, meta_k: float = 0) -> tuple[int, float]:
        payload = self.n_blocks * self.block_size
        return payload, payload + meta_k * self.grid**self.sym_modes

    def to_dense(self) -> np.ndarray:
        """Assemble the dense tensor this store represents (storage.py:525-536)."""
        b = self.block_dim
        out = np.empty(self.dims, dtype=np.float64, order="F")
        tail = tuple(slice(None) for _ in self.tail_dims)
        for key in itertools.product(range(self.grid), repeat=self.sym_modes):
            sl = tuple(slice(i * b, (i + 1) * b) for i in key) + tail
            out[sl] = self.partial_block_at(key)
        return out


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

    def block_at(self, idx: MultiIndex) -> np.ndarray:
        return self.partial_block_at(idx)


def packed_payload(a) -> np.ndarray:
    """Packed payload of any BCSS-like object: ours, or the reference's
    ``BcssTensor`` (blocks dict keyed by sorted tuples)."""
    if isinstance(a, PartialSymTensor):
        return a.payload
    grid = a.n // a.b
    return np.concatenate([
        np.asarray(a.blocks[key], dtype=np.float64).reshape(-1, order="F")
        for key in hypertriangle_iter(grid, a.order)
    ])
