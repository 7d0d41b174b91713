"""Randomized parity sweep (dev tool): random shapes through every execution
mode - device run, pipelined host run (mirrored order, cascade when chosen),
pageable staging, reuse=False, a workspace limit that forces waves, shard
plans over random unit subsets (gathered top-level rows), and the S5 helper
split (top-level plan, then start plans over a random child subset) - against
the numpy oracle (rel. Frobenius <= 1e-12; partial plans on their own blocks).

usage: python tools/fuzz.py [cases] [seed]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs
from oracle import bcss_oracle as orc
from paper_1301_7744_b200.dense import symmetrize_bcss_device

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
bad = 0
done = 0
while done < cases:
    m = int(rng.integers(2, 7))
    ba = int(rng.choice([1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 18, 20, 21, 22, 24, 25, 27, 28, 30, 32, 33, 36, 44, 48, 64] if m <= 3 else [1, 2, 4, 5, 6, 7, 8, 9, 10, 12, 14, 16]))
    bc = int(rng.choice([1, 2, 3, 4, 5, 6, 8, 12, 16] if m <= 4 else [1, 2, 3, 4, 6, 8]))
    nbar = int(rng.integers(1, {2: 9, 3: 7, 4: 5, 5: 4, 6: 3}[m] if ba < 36 else 4))
    pbar = int(rng.integers(1, {2: 9, 3: 7, 4: 5, 5: 4, 6: 3}[m]))
    n, p = ba * nbar, bc * pbar
    if orc.bcss_flops(m, n, p, ba, bc) > 2e9:  # keep the numpy oracle fast
        continue
    done += 1
    # half of the cases keep the fast kernels on shapes whose few columns per
    # key would send them to the generic kernel (the product's own rule)
    if rng.random() < 0.5:
        os.environ["BCSS_FORCE_FAST"] = "1"
    else:
        os.environ.pop("BCSS_FORCE_FAST", None)
    a = orc.random_bcss_packed(m, n, ba, int(rng.integers(1 << 30)))
    x = rng.standard_normal((p, n))
    want = orc.sttsm_bcss_packed(a, x, m, n, ba, bc)
    modes = {}
    plan = bs.SttsmPlan(m, n, p, ba, bc)
    c = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
    plan.run(torch.from_numpy(a).cuda(), torch.from_numpy(x).cuda(), c)
    torch.cuda.synchronize()
    modes["device"] = c.cpu().numpy()
    plan.close()
    waves = int(rng.integers(2, 5))
    plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=waves)
    ch = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64).pin_memory()
    plan.run_host(torch.from_numpy(a).pin_memory().numpy(), torch.from_numpy(x).pin_memory().numpy(), ch.numpy())
    modes["pipelined"] = ch.numpy().copy()
    cp = np.full(plan.c_elems, np.nan)
    plan.run_host(a, x, cp)
    modes["pageable"] = cp
    plan.close()
    # symmetric upload: on the (rounding-symmetric) input within 1e-12, and on
    # an exactly symmetrized copy bit for bit equal to the full upload
    plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=waves, symmetric_upload=True)
    ch = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64).pin_memory()
    plan.run_host(torch.from_numpy(a).pin_memory().numpy(), torch.from_numpy(x).pin_memory().numpy(), ch.numpy())
    modes["symmetric"] = ch.numpy().copy()
    a_ex = torch.from_numpy(a).cuda()
    symmetrize_bcss_device(a_ex, m, n, ba)
    a_ex = a_ex.cpu().pin_memory()
    ch.fill_(float("nan"))
    plan.run_host_async(a_ex.numpy(), torch.from_numpy(x).pin_memory().numpy(), ch.numpy())
    plan.wait()
    full_p = bs.SttsmPlan(m, n, p, ba, bc, pipeline=waves)
    cf = torch.full((full_p.c_elems,), float("nan"), dtype=torch.float64).pin_memory()
    full_p.run_host(a_ex.numpy(), torch.from_numpy(x).pin_memory().numpy(), cf.numpy())
    if not np.array_equal(ch.numpy(), cf.numpy()):
        bad += 1
        print(f"MISMATCH symmetric-vs-full bitwise m={m} n={n} p={p} ba={ba} bc={bc}", flush=True)
    full_p.close()
    plan.close()
    plan = bs.SttsmPlan(m, n, p, ba, bc, reuse=False)
    c = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
    plan.run(torch.from_numpy(a).cuda(), torch.from_numpy(x).cuda(), c)
    torch.cuda.synchronize()
    modes["noreuse"] = c.cpu().numpy()
    plan.close()
    full = bs.SttsmPlan(m, n, p, ba, bc)
    ws = full.workspace_bytes
    full.close()
    if ws > 0 and pbar > 1:
        try:
            plan = bs.SttsmPlan(m, n, p, ba, bc, workspace_limit=max(1, ws // 2))
            c = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
            plan.run(torch.from_numpy(a).cuda(), torch.from_numpy(x).cuda(), c)
            torch.cuda.synchronize()
            modes["waves"] = c.cpu().numpy()
            plan.close()
        except MemoryError:
            pass  # a single unit does not fit half the workspace
    blk = bc**m
    partial = {}
    # shard plan over a random subset of top-level units
    units = sorted(int(u) for u in rng.choice(pbar, size=int(rng.integers(1, pbar + 1)), replace=False))
    plan = bs.SttsmPlan(m, n, p, ba, bc, units=units)
    c = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64, device="cuda")
    plan.run(torch.from_numpy(a).cuda(), torch.from_numpy(x).cuda(), c)
    torch.cuda.synchronize()
    partial["shard"] = (c.cpu().numpy(), plan.c_block_ranks())
    plan.close()
    # helper split of one unit: T(m-1)[u] by a stop-level plan, children subset below
    u = int(rng.integers(0, pbar))
    kids = sorted(int(j) for j in rng.choice(u + 1, size=int(rng.integers(1, u + 2)), replace=False))
    top = bs.SttsmPlan(m, n, p, ba, bc, units=[u], stop_level=m - 1)
    t = torch.empty(top.c_elems, dtype=torch.float64, device="cuda")
    top.run(torch.from_numpy(a).cuda(), torch.from_numpy(x).cuda(), t)
    top.close()
    plan = bs.SttsmPlan(m, n, p, ba, bc, start_level=m - 1, start_calls=[(u,)], start_children=kids)
    c = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64, device="cuda")
    plan.run(t, torch.from_numpy(x).cuda(), c)
    torch.cuda.synchronize()
    partial["helper"] = (c.cpu().numpy(), plan.c_block_ranks())
    plan.close()
    for k, (v, ranks) in partial.items():
        idx = np.concatenate([np.arange(r * blk, (r + 1) * blk) for r in ranks]) if len(ranks) else np.zeros(0, int)
        err = orc.rel_frobenius(v[idx], want[idx]) if len(idx) else 0.0
        if not (err <= 1e-12):
            bad += 1
            print(f"MISMATCH {k} m={m} n={n} p={p} ba={ba} bc={bc}: rel {err:.3e}", flush=True)
    for k, v in modes.items():
        err = orc.rel_frobenius(v, want)
        if not (err <= 1e-12):
            bad += 1
            print(f"MISMATCH {k} m={m} n={n} p={p} ba={ba} bc={bc}: rel {err:.3e}", flush=True)
print(f"fuzz: {done} cases, {bad} mismatches")
