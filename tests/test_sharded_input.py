"""Multi-GPU host input: every rank uploads only its
pieces of A over its own PCIe link and the pieces reach the other GPUs by
broadcast, chunk events gating the top level (bcss_sttsm_run_gated).

CPU: the piece table covers A exactly once, balances the bytes, lets the
front of A arrive first, and every rank of a 2-rank gloo group derives the
same table.  GPU: a gated run is bit-identical to the plain run (one
process), and two processes sharing the one B200 - each holding and
uploading only its pieces, gloo broadcasting them - reproduce the single
plan's C bit for bit (the ranks' kernels never wait on each other).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1301_7744_b200 as bs
from paper_1301_7744_b200.distributed import (chunk_elems, chunk_ready_piece, input_pieces,
                                              partition_units, unit_flops)

CFGS = [(4, 512, 256, 32, 32), (3, 512, 512, 32, 32), (5, 96, 96, 8, 8), (4, 64, 64, 16, 16)]


@pytest.mark.parametrize("cfg", CFGS)
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_pieces_cover_a_once_and_balance(cfg, world):
    m, n, p, ba, bc = cfg
    total = sum(chunk_elems(m, n, ba))
    assert total == bs.simplex_count(n // ba, m) * ba**m
    pieces = input_pieces(m, n, ba, world)
    assert pieces[0][0] == 0 and pieces[-1][1] == total
    assert all(a[1] == b[0] for a, b in zip(pieces, pieces[1:]))
    assert all((hi - lo) % ba**m == 0 and hi > lo for lo, hi, _ in pieces)
    loads = [0] * world
    for lo, hi, r in pieces:
        loads[r] += hi - lo
    assert max(loads) <= 1.15 * total / world  # each PCIe link moves ~1/N of A
    # consecutive pieces belong to different ranks: the front of A arrives
    # over all links at once
    if world > 1:
        assert all(a[2] != b[2] for a, b in zip(pieces, pieces[1:]))
    ready = chunk_ready_piece(m, n, ba, pieces)
    ends = np.cumsum(chunk_elems(m, n, ba))
    for a, i in enumerate(ready):
        assert pieces[i][1] >= ends[a] and (i == 0 or pieces[i - 1][1] < ends[a])
    assert ready == sorted(ready)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _table_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, n, p, ba, bc = CFGS[0]
    mine = [(lo, hi) for lo, hi, r in input_pieces(m, n, ba, world) if r == rank]
    allm = [None] * world
    dist.all_gather_object(allm, mine)
    if rank == 0:
        flat = sorted(x for lst in allm for x in lst)
        q.put((flat, sum(chunk_elems(m, n, ba))))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_agree_on_piece_ownership():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_table_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(120)
        assert pr.exitcode == 0
    flat, total = q.get(timeout=10)
    assert flat[0][0] == 0 and flat[-1][1] == total
    assert all(a[1] == b[0] for a, b in zip(flat, flat[1:]))


# ---------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,kw", [((4, 64, 64, 16, 16), {}), ((3, 512, 512, 32, 32), {}),
                                    ((5, 48, 48, 8, 8), {"units": [1, 4]}),
                                    ((4, 64, 64, 16, 16), {"stop_level": 2}),
                                    ((3, 256, 256, 32, 32), {"pipeline": 3})])
def test_gated_run_is_bitwise_the_plain_run(cfg, kw):
    """One process: ShardedInput (world 1: chunked upload) + run_gated equals
    plan.run on resident inputs bit for bit (plain, shard, stop-level and
    pipelined/mirrored plans)."""
    from paper_1301_7744_b200.distributed import ShardedInput
    from paper_1301_7744_b200.generate import random_bcss_device, random_matrix_device

    m, n, p, ba, bc = cfg
    a = random_bcss_device(m, n, ba, 5)
    x = random_matrix_device(p, n, 6)
    plan = bs.SttsmPlan(m, n, p, ba, bc, **kw)
    ref = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64, device="cuda")
    plan.run(a, x, ref)
    shard = ShardedInput(m, n, ba, 0, 1, "cuda")
    shard.fill_from(a.cpu())
    a2 = torch.full_like(a, float("nan"))
    got = torch.full_like(ref, float("nan"))
    evs = shard.start(a2)
    plan.run_gated(a2, x, got, evs)
    torch.cuda.synchronize()
    assert torch.equal(a2, a)
    if "units" in kw:
        r = torch.as_tensor(plan.c_block_ranks(), device="cuda")
        blk = bc**m
        assert torch.equal(got.view(-1, blk)[r], ref.view(-1, blk)[r])
    else:
        assert torch.equal(got, ref)
    plan.close()


def _gpu_worker(rank, world, port, cfg, out):
    from paper_1301_7744_b200.distributed import OwnBlocksDownload, ShardedInput
    from paper_1301_7744_b200.generate import random_bcss_device, random_matrix_device

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    m, n, p, ba, bc = cfg
    a_full = random_bcss_device(m, n, ba, 9).cpu()  # stands in for the caller's host A
    x = random_matrix_device(p, n, 10)
    shard = ShardedInput(m, n, ba, rank, world, "cuda")
    shard.fill_from(a_full)
    del a_full  # from here on this rank holds only its own pieces
    parts = partition_units(unit_flops(m, n, p, ba, bc), world)
    plan = bs.SttsmPlan(m, n, p, ba, bc, units=parts[rank])
    a = torch.full((plan.a_elems,), float("nan"), dtype=torch.float64, device="cuda")
    c = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64, device="cuda")
    evs = shard.start(a)
    plan.run_gated(a, x, c, evs)
    down = OwnBlocksDownload(plan.c_block_ranks(), bc**m)
    down.start(c, torch.cuda.current_stream())
    torch.cuda.synchronize()
    np.save(out / f"rank{rank}_c.npy", down.host[:down.elems].numpy())
    np.save(out / f"rank{rank}_ranks.npy", np.sort(plan.c_block_ranks()))
    np.save(out / f"rank{rank}_hostbytes.npy", np.array([shard.host_bytes]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [(4, 64, 64, 16, 16), (3, 256, 256, 32, 32)])
def test_two_process_sharded_upload_reproduces_single_plan(cfg, tmp_path):
    from paper_1301_7744_b200.generate import random_bcss_device, random_matrix_device

    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, cfg, tmp_path)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(300)
        assert pr.exitcode == 0
    m, n, p, ba, bc = cfg
    a = random_bcss_device(m, n, ba, 9)
    x = random_matrix_device(p, n, 10)
    plan = bs.SttsmPlan(m, n, p, ba, bc)
    ref = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
    plan.run(a, x, ref)
    torch.cuda.synchronize()
    ref = ref.cpu().numpy().reshape(-1, bc**m)
    seen = np.zeros(ref.shape[0], bool)
    a_bytes = 8 * a.numel()
    for r in range(2):
        ranks = np.load(tmp_path / f"rank{r}_ranks.npy")
        got = np.load(tmp_path / f"rank{r}_c.npy").reshape(-1, bc**m)
        assert np.array_equal(got, ref[ranks])
        seen[ranks] = True
        assert np.load(tmp_path / f"rank{r}_hostbytes.npy")[0] <= 0.6 * a_bytes  # about half of A each
    assert seen.all()
