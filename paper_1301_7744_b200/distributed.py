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
    """(owners, subs, groups) of scheme S5 with release times.

    Owners: LPT over the owner costs (top-level rows of unit u plus its
    level-(m-2) calls (i, u), i <= u).  A subtree call (i, u) is *released*
    when the rank owning u finishes its owner plan (modelled as that rank's
    owner flops), so the subtrees are list-scheduled by release time: each
    call goes to the rank where it would finish first, max(free, release) +
    cost.  groups[r] = [(lo, hi, src_ranks)]: subs[r][lo:hi] run as one
    subtree plan once the owners in src_ranks have finished; consecutive
    calls share a group unless the later one would otherwise wait.  No
    global barrier separates the phases - a rank starts its first group as
    soon as its own owner plan and that group's sources are done (config 5 at
    8 GPUs: the barrier-separated schedule modelled 0.64 efficiency, this one
    0.87 - bounded by the largest owner).
    """
    pbar = p // b_c
    if m < 3:  # no level below m-2 to hand out: plain S1
        parts = partition_units(unit_flops(m, n, p, b_a, b_c, reuse), world)
        return parts, [[] for _ in range(world)], [[] for _ in range(world)]
    owner_cost = []
    for u in range(pbar):
        pl = SttsmPlan(m, n, p, b_a, b_c, reuse=reuse, units=[u], stop_level=m - 2)
        owner_cost.append(pl.stats()["flops"])
        pl.close()
    loads = [0] * world
    owners: list[list[int]] = [[] for _ in range(world)]
    owner_of = {}
    for u in sorted(range(pbar), key=lambda q: (-owner_cost[q], q)):
        r = min(range(world), key=lambda q: (loads[q], q))
        owners[r].append(u)
        owner_of[u] = r
        loads[r] += owner_cost[u]
    release = {u: loads[owner_of[u]] for u in range(pbar)}
    # subtree cost depends only on i (the row block) for fixed shapes
    sub_cost = {}
    for i in range(pbar):
        pl = SttsmPlan(m, n, p, b_a, b_c, reuse=reuse, start_level=m - 2, start_calls=[(i, pbar - 1)])
        sub_cost[i] = pl.stats()["flops"]
        pl.close()
    calls = sorted(((i, u) for u in range(pbar) for i in range(u + 1)),
                   key=lambda c: (release[c[1]], -sub_cost[c[0]], c))
    free = list(loads)
    subs: list[list[tuple]] = [[] for _ in range(world)]
    starts: list[list[int]] = [[] for _ in range(world)]
    for c in calls:
        rel, cost = release[c[1]], sub_cost[c[0]]
        r = min(range(world), key=lambda q: (max(free[q], rel) + cost, free[q], q))
        st = max(free[r], rel)
        subs[r].append(c)
        starts[r].append(st)
        free[r] = st + cost
    groups: list[list[tuple]] = [[] for _ in range(world)]
    for r in range(world):
        lo = 0
        for j in range(1, len(subs[r]) + 1):
            # a call that would start later than the group's first call because it
            # waits for its owner (not for the calls before it) opens a new group
            if j == len(subs[r]) or release[subs[r][j][1]] > max(starts[r][lo], loads[r]):
                src = sorted({owner_of[c[1]] for c in subs[r][lo:j]})
                groups[r].append((lo, j, src))
                lo = j
    return [sorted(o) for o in owners], subs, groups


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
    """One rank's share of the scheme-S5 schedule, with its plans, buffers and
    exchange list built once; ``run`` executes one full step (phase 1,
    T(m-2) exchange, phase 2) asynchronously on the current stream / NCCL.

    Phase 2 is one subtree plan per release group (``s5_groups``).  With the
    fused exchange there is no barrier between the phases: every rank records
    a CUDA IPC event after its owner plan, and each group's plan waits on the
    events of the owners it reads from, so a rank whose owner work is short
    starts its subtrees while the long owners still run."""

    def __init__(self, m: int, n: int, p: int, b_a: int, b_c: int, rank: int, world: int, device,
                 reuse: bool = True, group=None, compute=_gpu_compute, exchange: str = "nccl"):
        import torch

        self.m, self.rank, self.world, self.group, self.compute = m, rank, world, group, compute
        if exchange not in ("nccl", "peer", "auto"):
            raise ValueError(f"exchange must be 'nccl', 'peer' or 'auto', not {exchange!r}")
        self.exchange = exchange
        owners, subs, groups = s5_groups(m, n, p, b_a, b_c, world, reuse)
        self.owners, self.subs, self.groups = owners, subs, groups[rank]
        owner_of = {u: r for r in range(world) for u in owners[r]}
        self.plan_o = (SttsmPlan(m, n, p, b_a, b_c, reuse=reuse, units=owners[rank], stop_level=m - 2)
                       if owners[rank] else None)
        # one subtree plan per release group: slots subs[rank][lo:hi] of the receive buffer
        self.plans_s = [SttsmPlan(m, n, p, b_a, b_c, reuse=reuse, start_level=m - 2,
                                  start_calls=subs[rank][lo:hi]) for lo, hi, _ in self.groups]
        self._ev_own, self._ev_peer = None, {}
        probe = SttsmPlan(m, n, p, b_a, b_c, reuse=reuse, start_level=m - 2, start_calls=[(0, 0)])
        self.slice = probe.a_elems
        probe.close()
        # call order of every owner's T(m-2) buffer (deterministic, no communication)
        order = {}
        for r in range(world):
            if owners[r]:
                pl = SttsmPlan(m, n, p, b_a, b_c, reuse=reuse, units=owners[r], stop_level=m - 2)
                order[r] = {c: i for i, c in enumerate(pl.level_calls(m - 2))}
                pl.close()
        self.t2 = None  # owner output buffer (NCCL exchange only; the fused exchange stores to the slots)
        self._buf, self._peers = None, []
        if exchange in ("peer", "auto"):
            # fused exchange: every rank's receive buffer is opened by the others
            # (CUDA IPC); the owner's level-(m-2) kernel stores each call's
            # T(m-2) slice straight into its assignee's slot (NVLink peer stores).
            # "auto" falls back to NCCL send/recv if any rank cannot map a peer.
            import torch.distributed as dist

            ok, err = True, ""
            solo = world == 1 or not dist.is_initialized()
            try:
                self._buf = DeviceBuffer(max(1, len(subs[rank])) * self.slice, device)
                handle = None if solo else self._buf.ipc_handle()
            except Exception as e:  # noqa: BLE001 - reported below / fallback
                ok, err, handle = False, str(e), None
            handles = [handle] * world
            if not solo:
                dist.all_gather_object(handles, handle, group=group)
            base = {}
            if ok and (solo or all(h is not None for h in handles)):
                try:
                    for r in range(world):
                        if r == rank:
                            base[r] = self._buf.ptr
                        elif subs[r]:
                            base[r] = open_peer(handles[r])
                            self._peers.append(base[r])
                except Exception as e:  # noqa: BLE001
                    ok, err = False, str(e)
            else:
                ok = False
            flags = [ok] * world
            if not solo:
                dist.all_gather_object(flags, ok, group=group)
            if all(flags) and not solo:
                # owner-done events: group g of an assignee waits on its sources' events
                try:
                    self._ev_own = torch.cuda.Event(interprocess=True)
                    ev_handle = self._ev_own.ipc_handle()
                except Exception as e:  # noqa: BLE001
                    ok, err, ev_handle = False, str(e), None
                ev_handles = [ev_handle] * world
                dist.all_gather_object(ev_handles, ev_handle, group=group)
                need = {q for _, _, src in self.groups for q in src if q != rank}
                try:
                    for q in need:
                        if ev_handles[q] is None:
                            raise RuntimeError(f"rank {q} has no owner event")
                        self._ev_peer[q] = torch.cuda.Event.from_ipc_handle(device, ev_handles[q])
                except Exception as e:  # noqa: BLE001
                    ok, err = False, str(e)
                flags = [ok] * world
                dist.all_gather_object(flags, ok, group=group)
            if all(flags):
                self.exchange = "peer"
                self.inp = self._buf.tensor
                self.dest = self.peer_destinations(subs, rank)
                if self.plan_o is not None:
                    self.plan_o.set_call_outputs([base[r] + 8 * self.slice * j for r, j in self.dest])
            elif exchange == "peer":
                raise RuntimeError(f"fused peer exchange unavailable on some rank: {err}")
            else:
                self.exchange = "nccl"
        if self.exchange != "peer":
            self.inp = torch.empty(max(1, len(subs[rank])) * self.slice, dtype=torch.float64, device=device)
            if self.plan_o is not None:
                self.t2 = torch.empty(self.plan_o.c_elems, dtype=torch.float64, device=device)
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
        full = SttsmPlan(m, n, p, b_a, b_c)
        self.c_elems = full.c_elems
        full.close()

    def peer_destinations(self, subs, rank) -> list[tuple[int, int]]:
        """(assignee rank, slot) of every call of this rank's owner plan, in the
        plan's level-(m-2) call order (the fused exchange's pointer table)."""
        if self.plan_o is None:
            return []
        where = {c: (r, j) for r in range(len(subs)) for j, c in enumerate(subs[r])}
        return [where[tuple(c)] for c in self.plan_o.level_calls(self.m - 2)]

    def plans(self):
        return ([self.plan_o] if self.plan_o is not None else []) + list(self.plans_s)

    def _run_groups(self, x, c, wait_peers: bool) -> None:
        import torch

        s = self.slice
        stream = torch.cuda.current_stream(x.device) if wait_peers else None
        for (lo, hi, src), pl in zip(self.groups, self.plans_s):
            if wait_peers:
                for q in src:
                    if q != self.rank:  # own owner work precedes on this stream
                        stream.wait_event(self._ev_peer[q])
            self.compute(pl, self.inp[lo * s:hi * s], x, c)

    def attach_torch_workspace(self, device=None) -> None:
        for pl in self.plans():
            pl.attach_torch_workspace(device)

    def run(self, a, x, c) -> None:
        import torch.distributed as dist

        s = self.slice
        if self.exchange == "peer":
            import torch

            multi = self.world > 1 and self._ev_own is not None
            if multi:
                # the previous step's subtree plans finished reading every receive
                # buffer before any owner overwrites one
                torch.cuda.synchronize()
                dist.barrier(group=self.group)
            stream = torch.cuda.current_stream(x.device)
            if self.plan_o is not None:  # writes every T(m-2) slice into its assignee's buffer
                # every call has a destination, so the output buffer is never touched
                if self.plan_o._ws is None:
                    self.plan_o.attach_torch_workspace(x.device)
                self.plan_o.run_ptr(a.data_ptr(), x.data_ptr(), self.inp.data_ptr(), stream.cuda_stream)
            if multi:
                self._ev_own.record(stream)
                dist.barrier(group=self.group)  # every owner event of this step is recorded (host only)
            self._run_groups(x, c, wait_peers=multi)
            return
        if self.plan_o is not None:
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
