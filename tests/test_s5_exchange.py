"""The fused S5 exchange (owner kernel stores T(m-2) slices straight into the
assignee's receive buffer): its destination table matches the NCCL send/recv
plan (CPU), and two processes sharing one GPU through CUDA IPC reproduce the
single-plan C bit for bit (GPU; the ranks' kernels never wait on each other,
synchronization is a host barrier)."""

import os
import socket

import numpy as np
import pytest

import paper_1301_7744_b200 as bs
from paper_1301_7744_b200.distributed import S5Runner

CFG = (4, 64, 64, 16, 16)


@pytest.mark.parametrize("world", [2, 3])
def test_peer_destinations_match_nccl_exchange(world):
    m, n, p, ba, bc = CFG
    runners = [S5Runner(m, n, p, ba, bc, r, world, "cpu") for r in range(world)]
    for r, run in enumerate(runners):
        if run.plan_o is None:
            continue
        dest = run.peer_destinations(run.subs, r)
        calls = [tuple(c) for c in run.plan_o.level_calls(m - 2)]
        assert len(dest) == len(calls)
        sends = {i: q for q, i in run.sends}
        local = {i: j for j, i in run.local}
        for i, (q, j) in enumerate(dest):
            assert run.subs[q][j] == calls[i]
            if q == r:
                assert local[i] == j
            else:
                assert sends[i] == q and (r, j) in runners[q].recvs


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out, cfg=CFG, force=False):
    import torch
    import torch.distributed as dist

    from paper_1301_7744_b200.generate import random_bcss_device, random_matrix_device

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    m, n, p, ba, bc = cfg
    a = random_bcss_device(m, n, ba, 7)
    x = random_matrix_device(p, n, 8)
    run = S5Runner(m, n, p, ba, bc, rank, world, x.device, exchange="peer", force_helper=force)
    assert run.exchange == "peer" and (not force or run.sched["helper"])
    run.attach_torch_workspace()
    c = torch.full((run.c_elems,), float("nan"), dtype=torch.float64, device="cuda")
    for _ in range(2):  # twice: buffers and tables are reused across steps
        run.run(a, x, c)
    torch.cuda.synchronize()
    ranks = run.c_block_ranks()
    blk = bc**m
    mine = {int(r): c[int(r) * blk:(int(r) + 1) * blk].cpu().numpy() for r in ranks}
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    if rank == 0:
        plan = bs.SttsmPlan(*cfg)
        want = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
        plan.run(a, x, want)
        want = want.cpu().numpy()
        got = np.full_like(want, np.nan)
        for part in parts:
            for r, v in part.items():
                got[r * blk:(r + 1) * blk] = v
        out.put(bool(np.array_equal(got, want)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,force", [(CFG, False), ((4, 64, 32, 16, 16), True)])
def test_fused_peer_exchange_two_processes_one_gpu(cfg, force):
    """force=True: rank 0 owns unit 1 and hands child 1 to rank 1 (helper): the
    T(m-1) peer copy, the helper's start plan and the cross-process event
    waits all run."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, cfg, force)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    assert q.get(timeout=10) is True
