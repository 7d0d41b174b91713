"""Predict the S5 multi-GPU schedule's strong scaling on ONE B200.

Every virtual rank's phase-1 (owner) plan and phase-2 (subtree) plan is timed
device-resident, one after the other, and the job is replayed from those
times: rank r runs its owner plan, then each release group's subtree plan
once its source owners are done (S5Runner gates the groups on the owners'
CUDA IPC events; no barrier between the phases).  For comparison the
barrier-separated model max(owner) + max(subtree) is printed too.  The
exchange itself is fused into the owners' kernels (peer stores over NVLink)
and is not modelled here.

usage: python tools/s5_timing.py CONFIG [WORLD ...]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs
from paper_1301_7744_b200.distributed import s5_groups

CFGS = {2: (3, 512, 512, 32, 32), 3: (4, 192, 192, 16, 16), 4: (5, 96, 96, 8, 8), 5: (4, 512, 256, 32, 32)}


def timed(plan, inp, X, out, reps):
    plan.attach_torch_workspace()
    plan.run(inp, X, out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        plan.run(inp, X, out)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    cfg = int(sys.argv[1])
    worlds = [int(w) for w in sys.argv[2:]] or [2, 4, 8]
    reps = 3 if cfg == 5 else 5
    m, n, p, ba, bc = CFGS[cfg]
    full = bs.SttsmPlan(m, n, p, ba, bc)
    A = torch.rand(full.a_elems, dtype=torch.float64, device="cuda") * 2 - 1
    X = torch.randn(p, n, dtype=torch.float64, device="cuda")
    C = torch.empty(full.c_elems, dtype=torch.float64, device="cuda")
    t1 = timed(full, A, X, C, reps)
    total = full.stats()["flops"]
    full.close()
    del C
    torch.cuda.empty_cache()
    print(json.dumps({"config": cfg, "t1_ms": round(t1, 3), "tflops_1": round(total / t1 / 1e9, 2)}), flush=True)
    for w in worlds:
        owners, subs, groups = s5_groups(m, n, p, ba, bc, w)
        t_o, t_s, t_g, fl = [], [], [], []
        for r in range(w):
            f = 0
            if owners[r]:
                pl = bs.SttsmPlan(m, n, p, ba, bc, units=owners[r], stop_level=m - 2)
                out = torch.empty(pl.c_elems, dtype=torch.float64, device="cuda")
                t_o.append(round(timed(pl, A, X, out, reps), 3))
                f += pl.stats()["flops"]
                pl.close()
                del out
            else:
                t_o.append(0.0)
            torch.cuda.empty_cache()
            tg = []
            for lo, hi, _ in groups[r]:
                pl = bs.SttsmPlan(m, n, p, ba, bc, start_level=m - 2, start_calls=subs[r][lo:hi])
                inp = torch.rand(pl.a_elems, dtype=torch.float64, device="cuda")
                out = torch.empty(pl.c_elems, dtype=torch.float64, device="cuda")
                tg.append(round(timed(pl, inp, X, out, reps), 3))
                f += pl.stats()["flops"]
                pl.close()
                del inp, out
                torch.cuda.empty_cache()
            t_g.append(tg)
            t_s.append(round(sum(tg), 3))
            fl.append(f)
        ends = []
        for r in range(w):
            t = t_o[r]
            for (lo, hi, src), tg in zip(groups[r], t_g[r]):
                t = max([t] + [t_o[q] for q in src]) + tg
            ends.append(round(t, 3))
        overlap = max(ends)
        barrier = max(t_o) + max(t_s)
        print(json.dumps({"world": w, "owners": owners, "n_subs": [len(s) for s in subs],
                          "owner_ms": t_o, "sub_ms": t_s,
                          "flop_balance": round(sum(fl) / w / max(fl), 4),
                          "job_ms_barrier": round(barrier, 3), "eff_barrier": round(t1 / w / barrier, 4),
                          "rank_end_ms": ends, "groups": [len(g) for g in groups],
                          "job_ms_gated": round(overlap, 3), "eff_gated": round(t1 / w / overlap, 4)}),
              flush=True)


if __name__ == "__main__":
    main()
