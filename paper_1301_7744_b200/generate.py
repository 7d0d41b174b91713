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

import itertools
import math

from .indexing import hypertriangle_iter, simplex_count


def _runs(key) -> tuple[int, ...]:
    """Run lengths of equal consecutive values of a sorted block index."""
    out, cur = [], 1
    for a, b in zip(key, key[1:]):
        if a == b:
            cur += 1
        else:
            out.append(cur)
            cur = 1
    out.append(cur)
    return tuple(out)


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
    # group the blocks that need symmetrizing by their repeated-index pattern
    by_pattern: dict[tuple[int, ...], list[int]] = {}
    for r, key in enumerate(hypertriangle_iter(grid, m)):
        runs = _runs(key)
        if max(runs) > 1:
            by_pattern.setdefault(runs, []).append(r)
    blocks = out.view(nblk, *([b] * m))  # torch axes are the F-order modes reversed
    for runs, ranks in by_pattern.items():
        groups, start = [], 0
        for ln in runs:
            if ln > 1:
                # modes start..start+ln-1 live on torch axes 1+(m-1-d)
                groups.append([1 + (m - 1 - d) for d in range(start, start + ln)])
            start += ln
        idx_all = torch.tensor(ranks, dtype=torch.long, device=device)
        for c0 in range(0, len(ranks), step):
            idx = idx_all[c0:c0 + step]
            x = blocks.index_select(0, idx)
            for axes in groups:
                acc = torch.zeros_like(x)
                perms = list(itertools.permutations(axes))
                for perm in perms:
                    order = list(range(m + 1))
                    for src, dst in zip(axes, perm):
                        order[src] = dst
                    acc += x.permute(order)
                x = acc / math.factorial(len(axes))
            blocks.index_copy_(0, idx, x)
    return out


def random_matrix_device(p: int, n: int, seed: int, device="cuda"):
    """X ~ N(0,1), p x n row-major (BASELINE.json configs)."""
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    return torch.randn(p, n, dtype=torch.float64, device=device, generator=g)
