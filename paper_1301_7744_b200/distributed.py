"""Multi-GPU sharding of BCSS sttsm: one process per GPU over torch.distributed.

The path partitions naturally: C's canonical blocks split into top-level
subtrees (units) ``jb_{m-1} = j`` of the reference's ``descend``
(/root/reference/pkg/src/blocksym/change_of_basis.py:269-283); each subtree
needs all of A and X but shares nothing else, so ranks compute disjoint C
blocks with no data-path collective.  The exchanges are input distribution
(``broadcast_inputs``: A and X once over NVLink by NCCL) and, when the caller
wants C on one rank, the gather of the disjoint blocks (``gather_c``).

Subtree costs grow with j, so units are assigned longest-processing-time
first (LPT) on their exact flop counts (scheme S1).
"""

from __future__ import annotations

import numpy as np

from .sttsm import SttsmPlan


def unit_flops(m: int, n: int, p: int, b_a: int, b_c: int, reuse: bool = True) -> list[int]:
    """Exact flops of every top-level subtree j = 0..p/b_c-1 (host only)."""
    out = []
    for j in range(p // b_c):
        plan = SttsmPlan(m, n, p, b_a, b_c, reuse=reuse, units=[j])
        out.append(plan.stats()["flops"])
        plan.close()
    return out


def partition_units(costs: list[int], world: int) -> list[list[int]]:
    """LPT: heaviest unit first onto the least-loaded rank (ties -> lower rank)."""
    loads = [0] * world
    parts: list[list[int]] = [[] for _ in range(world)]
    for j in sorted(range(len(costs)), key=lambda u: (-costs[u], u)):
        r = min(range(world), key=lambda q: (loads[q], q))
        parts[r].append(j)
        loads[r] += costs[j]
    return [sorted(p) for p in parts]


def shard_plan(m: int, n: int, p: int, b_a: int, b_c: int, rank: int, world: int,
               reuse: bool = True, **kw) -> SttsmPlan:
    """The plan of ``rank``: its LPT share of the top-level units."""
    parts = partition_units(unit_flops(m, n, p, b_a, b_c, reuse), world)
    return SttsmPlan(m, n, p, b_a, b_c, reuse=reuse, units=parts[rank], **kw)


def broadcast_inputs(a, x, src: int = 0, group=None) -> None:
    """Replicate A (packed) and X from ``src`` to every rank (in place)."""
    import torch.distributed as dist

    dist.broadcast(a, src, group=group)
    dist.broadcast(x, src, group=group)


def gather_c(c_local, own_ranks: np.ndarray, all_ranks: list[np.ndarray], block_elems: int,
             dst: int = 0, group=None):
    """Assemble C on ``dst`` from disjoint per-rank blocks.

    ``c_local``: this rank's full-size packed C buffer (only its own blocks
    valid); ``own_ranks``: the payload ranks it wrote; ``all_ranks``: every
    rank's list (deterministic from the partition, so no size exchange).
    Blocks travel packed and padded to the largest share (one all_gather).
    Returns the assembled C on ``dst`` and ``c_local`` elsewhere.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    blocks = c_local.view(-1, block_elems)
    cap = max(len(r) for r in all_ranks)
    send = torch.zeros(cap, block_elems, dtype=c_local.dtype, device=c_local.device)
    if len(own_ranks):
        idx = torch.as_tensor(own_ranks, dtype=torch.long, device=c_local.device)
        send[: len(own_ranks)] = blocks.index_select(0, idx)
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send, group=group)
    if me != dst:
        return c_local
    out = c_local.clone().view(-1, block_elems)
    for r in range(world):
        if len(all_ranks[r]):
            idx = torch.as_tensor(all_ranks[r], dtype=torch.long, device=c_local.device)
            out.index_copy_(0, idx, recv[r][: len(all_ranks[r])])
    return out.view(-1)


def sttsm_bcss_distributed(a, x, m: int, b_a: int, b_c: int, reuse: bool = True, dst: int | None = 0,
                           group=None):
    """Sharded sttsm on torch CUDA tensors replicated on every rank.

    Each rank computes its LPT share of C; with ``dst`` set, C is gathered
    there (returned on ``dst``; other ranks get their partial buffer).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    p, n = x.shape
    parts = partition_units(unit_flops(m, n, p, b_a, b_c, reuse), world)
    plans = [SttsmPlan(m, n, p, b_a, b_c, reuse=reuse, units=u) for u in parts]
    plan = plans[rank]
    c = torch.zeros(plan.c_elems, dtype=torch.float64, device=x.device)
    plan.run(a, x, c)
    if dst is None:
        return c
    all_ranks = [pl.c_block_ranks() for pl in plans]
    return gather_c(c, all_ranks[rank], all_ranks, b_c**m, dst=dst, group=group)
