"""Predict multi-GPU strong scaling on ONE B200: time every rank's S1 shard
plan (its LPT share of the top-level units) device-resident, one after the
other, and report max-over-ranks against the single-plan time.  The ranks of
S1 exchange nothing inside the timed region, so the modelled job time is the
slowest rank's plan (A/X broadcast happens before timing).

usage: python tools/shard_timing.py CONFIG [WORLD ...]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs
from paper_1301_7744_b200.distributed import partition_units, unit_flops

CFGS = {2: (3, 512, 512, 32, 32), 3: (4, 192, 192, 16, 16), 4: (5, 96, 96, 8, 8), 5: (4, 512, 256, 32, 32)}


def launch_profile(plan, A, X, C):
    plan.set_timing(True)
    plan.run(A, X, C)
    out = [(k, round(fl / 1e9, 3), round(ms, 4), round(fl / ms / 1e9, 2)) for k, fl, ms in plan.launch_times()]
    plan.set_timing(False)
    return out


def time_plan(plan, A, X, C, reps=5):
    plan.attach_torch_workspace()
    for _ in range(2):
        plan.run(A, X, C)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    best = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        plan.run(A, X, C)
        e.record()
        torch.cuda.synchronize()
        best.append(s.elapsed_time(e))
    best.sort()
    return best[len(best) // 2]


def main():
    cfg = int(sys.argv[1])
    worlds = [int(w) for w in sys.argv[2:]] or [2, 4, 8]
    m, n, p, ba, bc = CFGS[cfg]
    full = bs.SttsmPlan(m, n, p, ba, bc)
    A = torch.rand(full.a_elems, dtype=torch.float64, device="cuda") * 2 - 1
    X = torch.randn(p, n, dtype=torch.float64, device="cuda")
    C = torch.empty(full.c_elems, dtype=torch.float64, device="cuda")
    t1 = time_plan(full, A, X, C)
    print(json.dumps({"full_launches (k, gflop, ms, TF)": launch_profile(full, A, X, C)}), flush=True)
    full.close()
    costs = unit_flops(m, n, p, ba, bc)
    out = {"config": cfg, "t1_ms": round(t1, 4), "worlds": {}}
    for w in worlds:
        parts = partition_units(costs, w)
        ts, prof = [], []
        for r in range(w):
            pl = bs.SttsmPlan(m, n, p, ba, bc, units=parts[r])
            ts.append(round(time_plan(pl, A, X, C), 4))
            prof.append(launch_profile(pl, A, X, C))
            pl.close()
            torch.cuda.empty_cache()
        loads = [sum(costs[u] for u in part) for part in parts]
        out["worlds"][w] = {"rank_ms": ts, "max_ms": max(ts), "eff": round(t1 / w / max(ts), 4),
                            "flop_balance": round(sum(costs) / w / max(loads), 4),
                            "slowest_rank_launches (k, gflop, ms, TF)": prof[ts.index(max(ts))]}
        print(json.dumps({w: out["worlds"][w]}), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
