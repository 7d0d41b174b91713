"""Multi-rank host logic on CPU (world_size 2, gloo, 127.0.0.1): LPT unit
partition, per-rank C shards (the CPU oracle stands in for the GPU kernel),
and the gather of disjoint C blocks onto rank 0 must reproduce the
reference's C (golden)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1301_7744_b200 as bs
from conftest import GOLDEN
from oracle import bcss_oracle as orc
from paper_1301_7744_b200.distributed import gather_c, partition_units, unit_flops


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = np.load(GOLDEN / f"sttsm_{case}.npz")
    m, n, p, ba, bc = (int(v) for v in d["dims"])
    parts = partition_units(unit_flops(m, n, p, ba, bc), world)
    plans = [bs.SttsmPlan(m, n, p, ba, bc, units=u) for u in parts]
    all_ranks = [pl.c_block_ranks() for pl in plans]
    local = orc.sttsm_bcss_packed(d["A"], d["X"], m, n, ba, bc, units=parts[rank])
    out = gather_c(torch.from_numpy(local), all_ranks[rank], all_ranks, bc**m, dst=0)
    if rank == 0:
        q.put((orc.rel_frobenius(out.numpy(), d["C"]), [len(u) for u in parts]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["config1", "rbcss_m4_n12_b4", "small_m3_n8_p12_ba2_bc4"])
def test_two_rank_shard_and_gather(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(120)
        assert pr.exitcode == 0
    err, sizes = q.get(timeout=10)
    assert err <= 1e-15 and sum(sizes) > 0 and min(sizes) > 0


def test_lpt_partition_balances_config5():
    costs = unit_flops(4, 512, 256, 32, 32)
    assert sum(costs) == bs.bcss_flops(4, 512, 256, 32, 32)
    for world in (2, 4, 8):
        parts = partition_units(costs, world)
        assert sorted(u for p in parts for u in p) == list(range(8))
        loads = [sum(costs[u] for u in p) for p in parts]
        assert max(loads) >= sum(costs) / world
        if world == 2:
            assert max(loads) / (sum(costs) / world) < 1.05
