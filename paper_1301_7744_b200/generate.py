"""Seeded BCSS inputs generated directly in HBM.

``random_bcss_device`` restates the reference generator ``random_bcss``
(/root/reference/pkg/src/blocksym/generate.py:53-77) on the GPU: U(-1,1) per
canonical block, then each block is averaged over the permutations of every
group of modes whose block indices repeat (generate.py:41-50, 69-76), so the
represented tensor is symmetric to rounding without ever being dense.  The
random stream is torch's (Philox), not numpy's, so values differ from the
reference's for the same seed; parity tests therefore feed identical packed
payloads to both sides instead of regenerating.
"""

from __future__ import annotations

from .dense import symmetrize_bcss_device
from .indexing import simplex_count


def random_bcss_device(m: int, n: int, b: int, seed: int, device="cuda", chunk_bytes: int = 1 << 30):
    """Packed payload (float64 CUDA tensor) of a random symmetric BCSS tensor."""
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    grid = n // b
    nblk = simplex_count(grid, m)
    bs = b**m
    out = torch.empty(nblk * bs, dtype=torch.float64, device=device)
    step = max(1, chunk_bytes // (bs * 8))
    for s in range(0, nblk, step):  # chunked fill keeps the generator's peak small
        e = min(nblk, s + step)
        out[s * bs:e * bs].uniform_(-1.0, 1.0, generator=g)
    # average every block over its repeated-index mode groups (generate.py:41-50)
    return symmetrize_bcss_device(out, m, n, b, chunk_blocks=step)


def random_matrix_device(p: int, n: int, seed: int, device="cuda"):
    """X ~ N(0,1), p x n row-major (BASELINE.json configs)."""
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    return torch.randn(p, n, dtype=torch.float64, device=device, generator=g)
