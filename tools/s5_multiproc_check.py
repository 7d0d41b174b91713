"""Run the S5 runner (fused peer exchange, helpers, IPC-event gating) with W
processes sharing one GPU and check the assembled C bit for bit against the
single-plan result.  A correctness check of the multi-rank wiring (the ranks'
kernels never spin on each other: cross-rank order is stream waits on CUDA
IPC events, host barriers are gloo), not a timing.

usage: python tools/s5_multiproc_check.py WORLD m n p b_a b_c
"""
import json
import os
import socket
import sys

import numpy as np

sys.path.insert(0, ".")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, cfg, q):
    import torch
    import torch.distributed as dist

    import paper_1301_7744_b200 as bs
    from paper_1301_7744_b200.distributed import S5Runner
    from paper_1301_7744_b200.generate import random_bcss_device, random_matrix_device

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    m, n, p, ba, bc = cfg
    a = random_bcss_device(m, n, ba, 17)
    x = random_matrix_device(p, n, 18)
    run = S5Runner(m, n, p, ba, bc, rank, world, x.device, exchange="peer")
    run.attach_torch_workspace()
    c = torch.full((run.c_elems,), float("nan"), dtype=torch.float64, device="cuda")
    for _ in range(3):  # buffers, tables and events are reused across steps
        run.run(a, x, c)
    torch.cuda.synchronize()
    blk = bc**m
    ranks = run.c_block_ranks()
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
        q.put({"world": world, "cfg": cfg, "helpers": {str(k): v for k, v in run.sched["helper"].items()},
               "groups": [len(g) for g in run.sched["groups"]], "exchange": run.exchange,
               "bitwise_equal": bool(np.array_equal(got, want))})
    dist.barrier()
    dist.destroy_process_group()


def main():
    import torch.multiprocessing as mp

    world = int(sys.argv[1])
    cfg = tuple(int(v) for v in sys.argv[2:7])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=900)
    codes = [pr.exitcode for pr in procs]
    res = q.get(timeout=10) if all(c == 0 for c in codes) else {"exitcodes": codes}
    print(json.dumps(res))
    sys.exit(0 if res.get("bitwise_equal") else 1)


if __name__ == "__main__":
    main()
