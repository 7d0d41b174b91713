"""Multi-GPU sharding of BCSS sttsm: one process per GPU over torch.distributed.

The path partitions naturally: C's canonical blocks split into top-level
subtrees (units) ``jb_{m-1} = j`` of the reference's ``descend``
(/root/reference/pkg/src/blocksym/change_of_basis.py:269-283); each subtree
needs all of A and X but shares nothing else, so ranks compute disjoint C
blocks with no data-path collective.  The exchanges are input distribution
(``broadcast_inputs``: A and X once over NVLink by NCCL) and, when the caller
wants C on one rank, the gather of the disjoint blocks (``gather_c``).

Subtree costs grow with j, so units are assigned longest-processing-time
first (LPT) on their exact flop counts (scheme S1): no exchange
at all, but the largest subtree bounds the balance (config 5 at 8 GPUs: 0.66).

``s5_schedule`` / ``sttsm_bcss_s5`` implement SURVEY §8e scheme S5: the owner
of top-level unit u computes T(m-1)[u] and the level-(m-2) calls (i, u)
(stop-level partial plan); every level-(m-2) call is then a subtree unit,
LPT-assigned over ranks on top of the owners' loads, and its T(m-2) (e.g.
1.14 GB for config 5) moves owner -> assignee by NCCL point-to-point before
the assignee runs the levels below (start-call partial plan).  Modelled
balance: 1.0 / 1.0 / 0.997 / 0.898 for configs 2-5 at 8 GPUs.
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


def s5_schedule(m: int, n: int, p: int, b_a: int, b_c: int, world: int, reuse: bool = True):
    """(owners, subs): owners[r] = top-level units rank r computes down to level
    m-2; subs[r] = level-(m-2) calls (i, u) whose subtrees rank r computes, in
    execution order.  Deterministic, so every rank derives the same schedule
    without talking.  See ``s5_groups`` for the release-time model."""
    owners, subs, _ = s5_groups(m, n, p, b_a, b_c, world, reuse)
    return owners, subs


def s5_groups(m: int, n: int, p: int, b_a: int, b_c: int, world: int, reuse: bool = True):
    """(owners, subs, groups) of scheme S5 without helpers; groups[r] =
    [(lo, hi, source ranks)] (see ``s5_tasks``)."""
    sc = s5_tasks(m, n, p, b_a, b_c, world, reuse, helpers=False)
    groups = [[(lo, hi, sorted({q for q, _ in src})) for lo, hi, src in g] for g in sc["groups"]]
    return sc["owners"], sc["subs"], groups


# modelled rates of the schedule (flop/s of the level kernels, B/s of an
# NVLink peer copy) - only their ratio matters: the T(m-1) transfer delay
RATE_FLOPS = 34e12
RATE_NVLINK = 600e9


def s5_tasks(m: int, n: int, p: int, b_a: int, b_c: int, world: int, reuse: bool = True,
             helpers: bool = True, force_helper: bool = False) -> dict:
    """Task schedule of scheme S5 (release times, optional helpers).

    Owners: LPT over the owner costs (top-level rows of unit u plus its
    level-(m-2) calls (i, u), i <= u).  **Helpers**: an owner of a single unit
    whose load exceeds the ideal share hands some of its level-(m-2) children
    to the least-loaded rank, which receives T(m-1)[u] by an NVLink peer copy
    after the owner's top level and computes those children from it (a start
    plan with a child subset); the owner computes the rest.  A subtree call
    (i, u) is *released* when the task producing its T(m-2) ends; the calls
    are list-scheduled by release time (each to the rank where it would
    finish first), and a rank's calls form release groups, one subtree plan
    each, which wait only on their sources' completion events.

    Times are modelled in flops (transfer = bytes x RATE_FLOPS / RATE_NVLINK).
    Returns {owners, helper: {u: (h, children)}, own_children: {u: children},
    help_of: {h: u}, subs, groups: [[(lo, hi, [(rank, "own"|"help")])]],
    model_end: per-rank modelled end}.  ``force_helper`` hands one child of
    the largest multi-child unit to another rank even when it does not pay
    (tests).
    """
    pbar = p // b_c
    if m < 3:  # no level below m-2 to hand out: plain S1
        parts = partition_units(unit_flops(m, n, p, b_a, b_c, reuse), world)
        return {"owners": parts, "helper": {}, "own_children": {}, "help_of": {},
                "subs": [[] for _ in range(world)], "groups": [[] for _ in range(world)], "model_end": None}
    owner_cost, top_cost = [], []
    for u in range(pbar):
        pl = SttsmPlan(m, n, p, b_a, b_c, reuse=reuse, units=[u], stop_level=m - 2)
        owner_cost.append(pl.stats()["flops"])
        pl.close()
    pl = SttsmPlan(m, n, p, b_a, b_c, reuse=reuse, units=[0], stop_level=m - 1)
    top = pl.stats()["flops"]  # every unit's top-level rows cost the same
    t_bytes = pl.c_elems * 8   # T(m-1) of one unit
    pl.close()
    lvl = [(owner_cost[u] - top) / (u + 1) for u in range(pbar)]  # per level-(m-2) call of unit u
    loads = [0.0] * world
    owners: list[list[int]] = [[] for _ in range(world)]
    owner_of = {}
    for u in sorted(range(pbar), key=lambda q: (-owner_cost[q], q)):
        r = min(range(world), key=lambda q: (loads[q], q))
        owners[r].append(u)
        owner_of[u] = r
        loads[r] += owner_cost[u]
    sub_cost = {}
    for i in range(pbar):
        pl = SttsmPlan(m, n, p, b_a, b_c, reuse=reuse, start_level=m - 2, start_calls=[(i, pbar - 1)])
        sub_cost[i] = pl.stats()["flops"]
        pl.close()
    total = sum(owner_cost) + sum(sub_cost[i] for u in range(pbar) for i in range(u + 1))
    ideal = total / world
    transfer = t_bytes * RATE_FLOPS / RATE_NVLINK
    own_end = list(loads)                       # end of each rank's owner task
    help_end: dict[int, float] = {}             # rank -> end of its help task
    helper: dict[int, tuple] = {}
    own_children = {u: list(range(u + 1)) for u in range(pbar)}
    help_of: dict[int, int] = {}
    if helpers and world > 1:
        for r in sorted(range(world), key=lambda q: (-loads[q], q)):
            if len(owners[r]) != 1:
                continue
            u = owners[r][0]
            if u == 0 or (own_end[r] <= ideal and not (force_helper and not helper)):
                continue
            cands = [q for q in range(world) if q != r and q not in help_of and owner_of.get(u) != q
                     and not any(helper.get(v, (None,))[0] == q for v in helper)]
            cands = [q for q in cands if all(owner_of[v] != q for v in helper)]
            if not cands:
                continue
            h = min(cands, key=lambda q: (own_end[q], q))
            best = None
            for c in range(1, u + 1):  # children handed over (the largest indices)
                e_owner = own_end[r] - c * lvl[u]
                e_help = max(own_end[h], top + transfer) + c * lvl[u]
                val = max(e_owner, e_help)
                if best is None or val < best[0]:
                    best = (val, c, e_owner, e_help)
            val, c, e_owner, e_help = best
            if val >= own_end[r] and not (force_helper and not helper):
                continue
            kids = list(range(u + 1 - c, u + 1))
            helper[u] = (h, kids)
            own_children[u] = list(range(u + 1 - c))
            help_of[h] = u
            own_end[r] = e_owner
            help_end[h] = e_help
    # release time of call (i, u): end of the task producing its T(m-2)
    release, source = {}, {}
    for u in range(pbar):
        for i in own_children[u]:
            release[(i, u)] = own_end[owner_of[u]]
            source[(i, u)] = (owner_of[u], "own")
        if u in helper:
            h, kids = helper[u]
            for i in kids:
                release[(i, u)] = help_end[h]
                source[(i, u)] = (h, "help")
    calls = sorted(((i, u) for u in range(pbar) for i in range(u + 1)),
                   key=lambda c: (release[c], -sub_cost[c[0]], c))
    free = [max(own_end[r], help_end.get(r, 0.0)) for r in range(world)]
    subs: list[list[tuple]] = [[] for _ in range(world)]
    starts: list[list[float]] = [[] for _ in range(world)]
    for c in calls:
        rel, cost = release[c], sub_cost[c[0]]
        r = min(range(world), key=lambda q: (max(free[q], rel) + cost, free[q], q))
        st = max(free[r], rel)
        subs[r].append(c)
        starts[r].append(st)
        free[r] = st + cost
    groups: list[list[tuple]] = [[] for _ in range(world)]
    for r in range(world):
        lo = 0
        prod_end = max(own_end[r], help_end.get(r, 0.0))
        for j in range(1, len(subs[r]) + 1):
            # a call that would start later than the group's first call because it
            # waits for its producer (not for the calls before it) opens a new group
            if j == len(subs[r]) or release[subs[r][j]] > max(starts[r][lo], prod_end):
                src = sorted({source[c] for c in subs[r][lo:j]})
                groups[r].append((lo, j, src))
                lo = j
    return {"owners": [sorted(o) for o in owners], "helper": helper, "own_children": own_children,
            "help_of": help_of, "subs": subs, "groups": groups, "model_end": free, "ideal": ideal}


# ---- multi-GPU host input: sharded upload + NVLink broadcast ---------------------
#
# Every C block depends on all of A, so every GPU needs all of A; on one node
# the host -> device links are per GPU (PCIe Gen5 x16, ~55 GB/s each) while
# NVLink/NVSwitch moves ~700 GB/s per GPU.  So the packed A is cut into
# pieces of equal size (at block boundaries), dealt round-robin to the ranks;
# rank r holds and uploads only its pieces, and every piece reaches the other
# GPUs by one NCCL broadcast from its owner, in ascending order.  Consecutive
# pieces belong to different ranks, so all PCIe links work in parallel and
# the front of A - what the top level's first key groups read (a key of first
# index a reads the first-index chunks 0..a, io.py:53-55 order) - lands first
# on every GPU.  The plan's top level waits per key group on per-chunk events
# (bcss_sttsm_run_gated), so the compute overlaps the rest of the transfer.

def chunk_elems(m: int, n: int, b_a: int) -> list[int]:
    """Elements of A's first-index chunks a = 0..n/b_a-1 (packed order)."""
    from math import comb

    nbar = n // b_a
    return [comb(nbar - a + m - 2, m - 1) * b_a**m for a in range(nbar)]


def input_pieces(m: int, n: int, b_a: int, world: int, per_rank: int = 8, min_pieces: int = 32):
    """(lo, hi, owner) element ranges of packed A: max(per_rank*world,
    min_pieces) pieces of equal block counts, owner = piece index mod world."""
    from math import comb

    nbar = n // b_a
    blocks = comb(nbar + m - 1, m)
    q = max(1, min(blocks, max(per_rank * world, min_pieces)))
    blk = b_a**m
    cuts = [blocks * i // q for i in range(q + 1)]
    return [(cuts[i] * blk, cuts[i + 1] * blk, i % world) for i in range(q) if cuts[i + 1] > cuts[i]]


def chunk_ready_piece(m: int, n: int, b_a: int, pieces) -> list[int]:
    """For every first-index chunk a, the index of the piece after whose
    arrival (pieces arrive in order) all of chunk a is resident."""
    sizes = chunk_elems(m, n, b_a)
    out, end = [], 0
    for e in sizes:
        end += e
        out.append(next(i for i, (_, hi, _) in enumerate(pieces) if hi >= end))
    return out


class ShardedInput:
    """One rank's share of A for the multi-GPU host path.

    Holds (pinned) only the pieces this rank owns (``input_pieces``); ``start``
    uploads them into the device copy of A on a copy stream and enqueues, for
    every piece in ascending order, an NCCL broadcast from its owner on a
    communication stream, recording the event of first-index chunk a once
    its last piece is resident.  With one rank it is a chunked upload with
    the same per-chunk events.
    """

    def __init__(self, m: int, n: int, b_a: int, rank: int, world: int, device, group=None):
        import torch

        self.m, self.n, self.b_a, self.rank, self.world, self.group = m, n, b_a, rank, world, group
        self.device = torch.device(device)
        self.nbar = n // b_a
        self.pieces = input_pieces(m, n, b_a, world)
        self.chunk_done_after = chunk_ready_piece(m, n, b_a, self.pieces)
        self.mine = [i for i, (_, _, r) in enumerate(self.pieces) if r == rank]
        self.host_off = {}
        off = 0
        for i in self.mine:
            lo, hi, _ = self.pieces[i]
            self.host_off[i] = off
            off += hi - lo
        self.host = torch.empty(max(1, off), dtype=torch.float64, pin_memory=True)
        self.h2d = torch.cuda.Stream(device=self.device)
        self.comm = torch.cuda.Stream(device=self.device)
        self.up_ev = {i: torch.cuda.Event() for i in self.mine}
        self.chunk_ev = [torch.cuda.Event() for _ in range(self.nbar)]
        self._src = [r for _, _, r in self.pieces]
        if world > 1:
            import torch.distributed as dist

            ranks = dist.get_process_group_ranks(group) if group is not None else list(range(world))
            self._src = [ranks[r] for r in self._src]  # global ranks of the owners

    @property
    def host_bytes(self) -> int:
        return 8 * sum(self.pieces[i][1] - self.pieces[i][0] for i in self.mine)

    def fill_from(self, a_full) -> None:
        """Copy this rank's pieces out of a full packed A (numpy or torch, host)."""
        import torch

        src = torch.as_tensor(a_full).reshape(-1)
        for i in self.mine:
            lo, hi, _ = self.pieces[i]
            o = self.host_off[i]
            self.host[o:o + hi - lo].copy_(src[lo:hi])

    def start(self, a_dev, after=None) -> list:
        """Enqueue this step's uploads and broadcasts into ``a_dev`` (the
        device copy of packed A); returns the per-chunk events.  ``after``
        (a torch.cuda.Event) orders them behind earlier readers of ``a_dev``."""
        import torch

        if after is not None:
            self.h2d.wait_event(after)
            self.comm.wait_event(after)
        with torch.cuda.stream(self.h2d):
            for i in self.mine:
                lo, hi, _ = self.pieces[i]
                o = self.host_off[i]
                a_dev[lo:hi].copy_(self.host[o:o + hi - lo], non_blocking=True)
                self.up_ev[i].record(self.h2d)
        done = {}
        for a, i in enumerate(self.chunk_done_after):
            done.setdefault(i, []).append(a)
        with torch.cuda.stream(self.comm):
            for i, (lo, hi, r) in enumerate(self.pieces):
                if r == self.rank:
                    self.comm.wait_event(self.up_ev[i])
                if self.world > 1:
                    import torch.distributed as dist

                    work = dist.broadcast(a_dev[lo:hi], src=self._src[i], group=self.group, async_op=True)
                    work.wait()  # the comm stream waits for the collective (the host does not block)
                for a in done.get(i, ()):
                    self.chunk_ev[a].record(self.comm)
        return self.chunk_ev


class OwnBlocksDownload:
    """D2H of the C blocks one rank computed (runs of consecutive packed
    ranks) into a compact pinned buffer."""

    def __init__(self, ranks, blk_c: int):
        import torch

        r = np.sort(np.asarray(ranks, dtype=np.int64))
        self.runs = []  # (device element offset, host element offset, elements)
        h, i = 0, 0
        while i < len(r):
            j = i + 1
            while j < len(r) and r[j] == r[j - 1] + 1:
                j += 1
            self.runs.append((int(r[i]) * blk_c, h, (j - i) * blk_c))
            h += (j - i) * blk_c
            i = j
        self.host = torch.empty(max(1, h), dtype=torch.float64, pin_memory=True)
        self.elems = h

    def start(self, c_dev, stream) -> None:
        import torch

        with torch.cuda.stream(stream):
            for d, h, e in self.runs:
                self.host[h:h + e].copy_(c_dev[d:d + e], non_blocking=True)


def _gpu_compute(plan: SttsmPlan, inp, x, out) -> None:
    plan.run(inp, x, out)


class DeviceBuffer:
    """Device memory from the library's own cudaMalloc (so its CUDA IPC handle
    covers exactly this buffer), viewed as a float64 torch tensor."""

    def __init__(self, elems: int, device):
        import ctypes

        import torch

        from . import _native

        self._lib = _native.lib()
        ptr = ctypes.c_void_p()
        _native.check(self._lib.bcss_device_alloc(ctypes.c_size_t(max(1, elems) * 8), ctypes.byref(ptr)))
        self.ptr = int(ptr.value)
        self.__cuda_array_interface__ = {"shape": (max(1, elems),), "typestr": "<f8", "data": (self.ptr, False),
                                         "version": 3, "strides": None}
        self.tensor = torch.as_tensor(self, device=device)

    def ipc_handle(self) -> bytes:
        import ctypes

        from . import _native

        buf = ctypes.create_string_buffer(64)
        _native.check(self._lib.bcss_ipc_get_handle(ctypes.c_void_p(self.ptr), buf))
        return buf.raw

    def close(self) -> None:
        import ctypes

        if getattr(self, "ptr", 0):
            self.tensor = None
            self._lib.bcss_device_free(ctypes.c_void_p(self.ptr))
            self.ptr = 0


def open_peer(handle: bytes) -> int:
    """Device address (valid in this process) of another rank's buffer."""
    import ctypes

    from . import _native

    out = ctypes.c_void_p()
    _native.check(_native.lib().bcss_ipc_open_handle(ctypes.create_string_buffer(handle, 64), ctypes.byref(out)))
    return int(out.value)


class S5Runner:
    """One rank's share of the scheme-S5 schedule (``s5_tasks``), with its
    plans, buffers and exchange tables built once; ``run`` executes one full
    step asynchronously on the current stream.

    Tasks on a rank, in stream order:
      1. owner work - either one plan over its units down to level m-2, or,
         for an owner with a helper, the top-level plan (T(m-1)[u] into a
         local buffer, then an NVLink peer copy of it into the helper's
         receive buffer on a side stream) and a level-(m-2) plan over the
         children it keeps;
      2. help work - a level-(m-2) plan over the handed-over children, reading
         the received T(m-1)[u] once the owner's copy event fired;
      3. one subtree plan per release group.
    Every level-(m-2) plan stores each call's T(m-2) straight into its
    assignee's receive slot (fused exchange, CUDA IPC peer stores).  Tasks
    of different ranks are ordered by CUDA IPC events ("sent", "own",
    "help") that the waiting rank's stream waits on; host barriers run over
    a gloo group, so they never wait for GPU work.  ``exchange="nccl"`` (or a
    rank that cannot map its peers under "auto") uses the schedule without
    helpers and NCCL send/recv between the phases.
    """

    def __init__(self, m: int, n: int, p: int, b_a: int, b_c: int, rank: int, world: int, device,
                 reuse: bool = True, group=None, compute=_gpu_compute, exchange: str = "nccl",
                 helpers: bool = True, force_helper: bool = False):
        if exchange not in ("nccl", "peer", "auto"):
            raise ValueError(f"exchange must be 'nccl', 'peer' or 'auto', not {exchange!r}")
        self.m, self.n, self.p, self.b_a, self.b_c, self.reuse = m, n, p, b_a, b_c, reuse
        self.rank, self.world, self.group, self.compute, self.device = rank, world, group, compute, device
        probe = SttsmPlan(m, n, p, b_a, b_c, reuse=reuse, start_level=m - 2, start_calls=[(0, 0)])
        self.slice = probe.a_elems
        probe.close()
        full = SttsmPlan(m, n, p, b_a, b_c)
        self.c_elems = full.c_elems
        full.close()
        self._plans_all: list[SttsmPlan] = []
        self._peers: list[int] = []
        self._bufs: list[DeviceBuffer] = []
        if exchange in ("peer", "auto"):
            err = self._setup(True, helpers, force_helper)
            if err is None:
                self.exchange = "peer"
                return
            if exchange == "peer":
                raise RuntimeError(f"fused peer exchange unavailable on some rank: {err}")
            self._teardown()
        self._setup(False, False, False)
        self.exchange = "nccl"

    # ---- construction -----------------------------------------------------------
    def _plan(self, **kw) -> SttsmPlan:
        pl = SttsmPlan(self.m, self.n, self.p, self.b_a, self.b_c, reuse=self.reuse, **kw)
        self._plans_all.append(pl)
        return pl

    def _teardown(self) -> None:
        for pl in self._plans_all:
            pl.close()
        self._plans_all = []
        for ptr in self._peers:
            try:
                from . import _native
                import ctypes
                _native.lib().bcss_ipc_close_handle(ctypes.c_void_p(ptr))
            except Exception:  # noqa: BLE001 - best effort
                pass
        self._peers = []
        for b in self._bufs:
            b.close()
        self._bufs = []

    def _setup(self, peer: bool, helpers: bool, force_helper: bool):
        """Build plans and buffers; returns None or the reason peer mode failed."""
        import torch

        m, rank, world, device = self.m, self.rank, self.world, self.device
        sc = s5_tasks(self.m, self.n, self.p, self.b_a, self.b_c, world, self.reuse,
                      helpers=helpers and peer, force_helper=force_helper)
        self.sched = sc
        owners, subs = sc["owners"], sc["subs"]
        self.owners, self.subs, self.groups = owners, subs, sc["groups"][rank]
        owner_of = {u: r for r in range(world) for u in owners[r]}
        self.owner_of = owner_of
        mine = owners[rank]
        helped = [u for u in mine if u in sc["helper"]]
        # 1. owner work
        self.plan_o = self.plan_top = self.plan_lvl = None
        self.top_unit = helped[0] if helped else None
        if self.top_unit is not None:
            u = self.top_unit
            self.plan_top = self._plan(units=[u], stop_level=m - 1)
            self.plan_lvl = self._plan(start_level=m - 1, start_calls=[(u,)],
                                       start_children=sc["own_children"][u], stop_level=m - 2)
        elif mine:
            self.plan_o = self._plan(units=mine, stop_level=m - 2)
        # 2. help work
        self.help_unit = sc["help_of"].get(rank)
        self.plan_help = None
        if self.help_unit is not None:
            v = self.help_unit
            self.plan_help = self._plan(start_level=m - 1, start_calls=[(v,)],
                                        start_children=sc["helper"][v][1], stop_level=m - 2)
        # 3. subtree plans, one per release group: slots subs[rank][lo:hi]
        self.plans_s = [self._plan(start_level=m - 2, start_calls=subs[rank][lo:hi]) for lo, hi, _ in self.groups]
        where = {c: (r, j) for r in range(world) for j, c in enumerate(subs[r])}
        self.producers = [pl for pl in (self.plan_o, self.plan_lvl, self.plan_help) if pl is not None]
        self.t_top = None
        if self.plan_top is not None:
            self.t_top = torch.empty(self.plan_top.c_elems, dtype=torch.float64, device=device)
        self._ev_own = self._ev_sent = self._ev_help = None
        self._ev_peer: dict = {}
        self._host_group = None
        if not peer:
            # NCCL exchange: the owner plan writes T(m-2) locally, then send/recv
            self.inp = torch.empty(max(1, len(subs[rank])) * self.slice, dtype=torch.float64, device=device)
            self.t2 = (torch.empty(self.plan_o.c_elems, dtype=torch.float64, device=device)
                       if self.plan_o is not None else None)
            order = {}
            for r in range(world):
                if owners[r]:
                    pl = SttsmPlan(self.m, self.n, self.p, self.b_a, self.b_c, reuse=self.reuse,
                                   units=owners[r], stop_level=m - 2)
                    order[r] = {c: i for i, c in enumerate(pl.level_calls(m - 2))}
                    pl.close()
            self.local, self.sends, self.recvs = [], [], []  # (dst slot, src slot) / (peer, slot)
            for r in range(world):
                for j, c in enumerate(subs[r]):
                    q = owner_of[c[1]]
                    if q == rank and r == rank:
                        self.local.append((j, order[q][c]))
                    elif q == rank:
                        self.sends.append((r, order[q][c]))
                    elif r == rank:
                        self.recvs.append((q, j))
            self.exchange_bytes = 8 * self.slice * (len(self.sends) + len(self.recvs))
            return None
        # fused exchange: every rank's receive buffers are opened by the others
        import torch.distributed as dist

        solo = world == 1 or not dist.is_initialized()
        hg = None
        if not solo:
            # host-only barriers and handle swaps over the same ranks as `group`
            members = None if self.group is None else dist.get_process_group_ranks(self.group)
            hg = self._host_group = dist.new_group(ranks=members, backend="gloo")
        ok, err = True, ""
        handles = (None, None, None)
        try:
            inbuf = DeviceBuffer(max(1, len(subs[rank])) * self.slice, device)
            self._bufs.append(inbuf)
            self.inp = inbuf.tensor
            self.recv_top = None
            if self.plan_help is not None:  # T(m-1) of the helped unit arrives here
                rb = DeviceBuffer(self.plan_help.a_elems, device)
                self._bufs.append(rb)
                self.recv_top = rb
            if not solo:
                self._ev_own = torch.cuda.Event(interprocess=True)
                self._ev_sent = torch.cuda.Event(interprocess=True)
                self._ev_help = torch.cuda.Event(interprocess=True)
                handles = (inbuf.ipc_handle(), self.recv_top.ipc_handle() if self.recv_top else None,
                           (self._ev_own.ipc_handle(), self._ev_sent.ipc_handle(), self._ev_help.ipc_handle()))
        except Exception as e:  # noqa: BLE001 - reported / fallback
            ok, err, handles = False, str(e), (None, None, None)
        allh = [handles] * world
        if not solo:
            dist.all_gather_object(allh, handles, group=hg)
        base, top_dst = {rank: self.inp.data_ptr()} if ok else {}, None
        if ok:
            try:
                for r in range(world):
                    if r != rank and subs[r]:
                        if allh[r][0] is None:
                            raise RuntimeError(f"rank {r} has no receive buffer")
                        base[r] = open_peer(allh[r][0])
                        self._peers.append(base[r])
                if self.top_unit is not None:
                    h = sc["helper"][self.top_unit][0]
                    if solo:
                        top_dst = self.recv_top.ptr if h == rank else None
                    else:
                        if allh[h][1] is None:
                            raise RuntimeError(f"helper rank {h} has no T(m-1) buffer")
                        top_dst = open_peer(allh[h][1])
                        self._peers.append(top_dst)
                if not solo:
                    need = set()
                    for _, _, src in self.groups:
                        need |= {(q, tag) for q, tag in src if q != rank}
                    if self.help_unit is not None:
                        need.add((owner_of[self.help_unit], "sent"))
                    idx = {"own": 0, "sent": 1, "help": 2}
                    for q, tag in need:
                        self._ev_peer[(q, tag)] = torch.cuda.Event.from_ipc_handle(device, allh[q][2][idx[tag]])
            except Exception as e:  # noqa: BLE001
                ok, err = False, str(e)
        flags = [ok] * world
        if not solo:
            dist.all_gather_object(flags, ok, group=hg)
        if not all(flags):
            return err or "a peer rank could not map the exchange buffers"
        self.top_dst = top_dst
        for pl in self.producers:
            pl.set_call_outputs([base[r] + 8 * self.slice * j for r, j in
                                 (where[tuple(c)] for c in pl.level_calls(m - 2))])
        self.t2 = None
        self.local, self.sends, self.recvs = [], [], []
        self.exchange_bytes = 8 * self.slice * sum(1 for pl in self.producers for c in pl.level_calls(m - 2)
                                                   if where[tuple(c)][0] != rank)
        if self.plan_top is not None and sc["helper"][self.top_unit][0] != rank:
            self.exchange_bytes += 8 * self.plan_top.c_elems
        self._side = torch.cuda.Stream(device=device)
        self._ev_top = torch.cuda.Event()
        return None

    def peer_destinations(self, subs, rank) -> list[tuple[int, int]]:
        """(assignee rank, slot) of every call of this rank's owner plan, in the
        plan's level-(m-2) call order (the fused exchange's pointer table)."""
        if self.plan_o is None:
            return []
        where = {c: (r, j) for r in range(len(subs)) for j, c in enumerate(subs[r])}
        return [where[tuple(c)] for c in self.plan_o.level_calls(self.m - 2)]

    def plans(self):
        return [pl for pl in (self.plan_o, self.plan_top, self.plan_lvl, self.plan_help) if pl is not None] + \
            list(self.plans_s)

    def attach_torch_workspace(self, device=None) -> None:
        for pl in self.plans():
            pl.attach_torch_workspace(device)

    # ---- one step ---------------------------------------------------------------
    def _run_groups(self, x, c, wait_peers: bool) -> None:
        import torch

        s = self.slice
        stream = torch.cuda.current_stream(x.device) if wait_peers else None
        for (lo, hi, src), pl in zip(self.groups, self.plans_s):
            if wait_peers:
                for q, tag in src:
                    if q != self.rank:  # own producer work precedes on this stream
                        stream.wait_event(self._ev_peer[(q, tag)])
            self.compute(pl, self.inp[lo * s:hi * s], x, c)

    def _run_ptr(self, pl: SttsmPlan, inp_ptr: int, x, out_ptr: int, stream, gate=None) -> None:
        if pl._ws is None:
            pl.attach_torch_workspace(x.device)
        if gate is not None:
            pl.run_gated_ptr(inp_ptr, x.data_ptr(), out_ptr, gate, stream.cuda_stream)
        else:
            pl.run_ptr(inp_ptr, x.data_ptr(), out_ptr, stream.cuda_stream)

    def run(self, a, x, c, gate_events=None) -> None:
        """One step on the current stream.  ``gate_events`` (one per
        first-index chunk of A, ``ShardedInput.start``): the plans that read A
        wait per top-level key group for the chunks they need instead of for
        all of A."""
        import torch.distributed as dist

        s = self.slice
        if self.exchange == "peer":
            import ctypes

            import torch

            from . import _native

            multi = self._host_group is not None
            hg = self._host_group
            if multi:
                # the previous step's readers of every receive buffer are done
                # before any rank overwrites one
                torch.cuda.synchronize()
                dist.barrier(group=hg)
            stream = torch.cuda.current_stream(x.device)
            # every call has a destination, so a producer's output buffer is never touched
            sink = self.inp.data_ptr()
            if self.plan_top is not None:
                self._run_ptr(self.plan_top, a.data_ptr(), x, self.t_top.data_ptr(), stream, gate_events)
                if self.top_dst is not None:  # T(m-1)[u] -> helper over NVLink, beside the level work
                    self._ev_top.record(stream)
                    self._side.wait_event(self._ev_top)
                    _native.check(_native.lib().bcss_copy_async(
                        ctypes.c_void_p(self.top_dst), ctypes.c_void_p(self.t_top.data_ptr()),
                        ctypes.c_size_t(8 * self.t_top.numel()), ctypes.c_void_p(self._side.cuda_stream)))
                    if multi:
                        self._ev_sent.record(self._side)
                    else:
                        stream.wait_stream(self._side)  # one process: the helper task follows on this stream
                self._run_ptr(self.plan_lvl, self.t_top.data_ptr(), x, sink, stream)
            elif self.plan_o is not None:
                self._run_ptr(self.plan_o, a.data_ptr(), x, sink, stream, gate_events)
            if multi:
                self._ev_own.record(stream)
                dist.barrier(group=hg)  # every "own"/"sent" event of this step is recorded
            if self.plan_help is not None:
                if multi:
                    stream.wait_event(self._ev_peer[(self.owner_of[self.help_unit], "sent")])
                self._run_ptr(self.plan_help, self.recv_top.ptr, x, sink, stream)
                if multi:
                    self._ev_help.record(stream)
            if multi:
                dist.barrier(group=hg)  # every "help" event of this step is recorded
            self._run_groups(x, c, wait_peers=multi)
            return
        if self.plan_o is not None:
            if gate_events is not None:
                import torch

                self.plan_o.run_gated(a, x, self.t2, gate_events, torch.cuda.current_stream(x.device))
            else:
                self.compute(self.plan_o, a, x, self.t2)
        for j, i in self.local:
            self.inp[j * s:(j + 1) * s].copy_(self.t2[i * s:(i + 1) * s])
        ops = [dist.P2POp(dist.isend, self.t2[i * s:(i + 1) * s], r, group=self.group) for r, i in self.sends]
        ops += [dist.P2POp(dist.irecv, self.inp[j * s:(j + 1) * s], q, group=self.group) for q, j in self.recvs]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        self._run_groups(x, c, wait_peers=False)

    def c_block_ranks(self) -> np.ndarray:
        if not self.plans_s:
            return np.zeros(0, dtype=np.int64)
        return np.concatenate([pl.c_block_ranks() for pl in self.plans_s])

    @property
    def flops(self) -> int:
        return sum(pl.stats()["flops"] for pl in self.plans())


def sttsm_bcss_s5(a, x, m: int, b_a: int, b_c: int, reuse: bool = True, dst: int | None = 0,
                  group=None, compute=_gpu_compute, exchange: str = "nccl"):
    """Scheme-S5 sharded sttsm (one rank per GPU).

    Phase 1: owned units down to level m-2 (T(m-2) of their calls into a
    local buffer).  Exchange: each level-(m-2) call's T(m-2) goes from its
    owner to the rank its subtree was assigned to (``exchange="nccl"``: NCCL
    send/recv; ``"peer"``: fused - the owner's kernel stores the slice straight
    into the assignee's receive buffer through a CUDA IPC mapping; local
    copies for self).  Phase 2: the assigned subtrees down to C.  With ``dst``
    set, C is gathered there.  ``compute(plan, inp, x, out)`` runs a plan
    (tests substitute a CPU stand-in).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    p, n = x.shape
    if m < 3:
        return sttsm_bcss_distributed(a, x, m, b_a, b_c, reuse=reuse, dst=dst, group=group)
    runner = S5Runner(m, n, p, b_a, b_c, rank, world, x.device, reuse=reuse, group=group, compute=compute,
                      exchange=exchange)
    c = torch.zeros(runner.c_elems, dtype=x.dtype, device=x.device)
    runner.run(a, x, c)
    if dst is None:
        return c
    all_ranks = []
    for r in range(world):
        sb = runner.subs[r]
        if sb:
            pl = SttsmPlan(m, n, p, b_a, b_c, reuse=reuse, start_level=m - 2, start_calls=sb)
            all_ranks.append(pl.c_block_ranks())
            pl.close()
        else:
            all_ranks.append(np.zeros(0, dtype=np.int64))
    return gather_c(c, all_ranks[rank], all_ranks, b_c**m, dst=dst, group=group)
