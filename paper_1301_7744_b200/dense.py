"""Dense baseline and symmetrization on the GPU.

``sttsm_dense_ttm_device`` is the reference's dense baseline
``sttsm_dense_ttm`` (/root/reference/pkg/src/blocksym/change_of_basis.py:141-154):
m successive mode products with the full X, ignoring symmetry and blocking,
flop count ``2 * sum_d p^{d+1} n^{m-d}`` (costs.py:145-171).  On B200 each mode
product is one cuBLAS DGEMM (torch.tensordot) — a *library* baseline, used to
reproduce the paper's BCSS-vs-Dense comparison on the
same GPU.  It needs the dense tensor (n^m doubles), so it only fits small n.

``symmetrize_bcss_device`` averages every canonical block of a packed BCSS
payload over the permutations of its repeated-index mode groups (native
kernel, csrc/symmetrize.cu), making the represented tensor exactly
symmetric — the blocked counterpart of the reference's ``symmetrize`` (change_of_basis.py:287-295), motivated at
PAPER.md:1461-1466 (diagonal blocks of C carry 1-ulp asymmetry).

``bcss_to_dense_device`` expands a packed payload to the dense tensor
(decompress, storage.py:525-536) on the GPU.
"""

from __future__ import annotations

import itertools
import math

from .indexing import canonicalize, hypertriangle_iter, hypertriangle_rank, simplex_count


def dense_flops(m: int, n: int, p: int) -> int:
    """dense_costs(m, n, p).flops (costs.py:145-171)."""
    return 2 * sum(p ** (d + 1) * n ** (m - d) for d in range(m))


def sttsm_dense_ttm_device(a_dense, x):
    """C = A x_0 X x_1 X ... x_{m-1} X on dense device tensors (cuBLAS DGEMMs).

    ``a_dense``: (n,)*m float64 CUDA tensor; ``x``: p x n.  Returns (p,)*m.
    Each step contracts the leading mode and appends the new one at the end,
    so after m steps the modes are back in order.
    """
    import torch

    c = a_dense
    for _ in range(a_dense.dim()):
        c = torch.tensordot(c, x, dims=([0], [1]))
    return c


def bcss_to_dense_device(packed, m: int, dim: int, b: int):
    """Dense (dim,)*m tensor represented by a packed payload (torch, on device).

    Dense index order is the tensor's mode order (mode 0 first); packed blocks
    are F-order, i.e. torch views with the modes reversed.
    """
    import torch

    g = dim // b
    blocks = packed.view(simplex_count(g, m), *([b] * m))
    out = torch.empty((dim,) * m, dtype=packed.dtype, device=packed.device)
    for idx in itertools.product(range(g), repeat=m):
        canon, mapping = canonicalize(idx)
        blk = blocks[hypertriangle_rank(canon, g)]           # torch axes = modes reversed
        stored_modes = blk.permute(*reversed(range(m)))      # axes = stored modes 0..m-1
        logical = stored_modes.permute(*mapping)             # logical mode d = stored mode mapping[d]
        sl = tuple(slice(i * b, (i + 1) * b) for i in idx)
        out[sl] = logical
    return out


def symmetrize_bcss_device(packed, m: int, dim: int, b: int, chunk_blocks: int = 256):
    """In-place symmetrization of the diagonal blocks of a packed payload (a
    float64 CUDA tensor): the native kernel ``bcss_symmetrize_blocks``
    (csrc/symmetrize.cu) averages every block whose key repeats an index over
    the permutations of each run of equal indices, on torch's current stream.
    ``chunk_blocks`` is accepted for compatibility and unused."""
    import ctypes

    import torch

    from . import _native

    if not (packed.is_cuda and packed.dtype == torch.float64 and packed.is_contiguous()):
        raise ValueError("symmetrize_bcss_device needs a contiguous float64 CUDA tensor")
    if packed.numel() != simplex_count(dim // b, m) * b**m:
        raise ValueError("payload size does not match (m, dim, b)")
    with torch.cuda.device(packed.device):
        stream = torch.cuda.current_stream(packed.device).cuda_stream
        _native.check(_native.lib().bcss_symmetrize_blocks(
            ctypes.c_void_p(packed.data_ptr()), m, dim, b, ctypes.c_void_p(stream)))
    return packed
