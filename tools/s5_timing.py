"""Predict the S5 multi-GPU schedule's strong scaling on ONE B200.

Every virtual rank's phase-1 (owner) plan and phase-2 (subtree) plan is timed
device-resident, one after the other, and the job is replayed from those
times: rank r runs its owner work (with a helper: top-level plan + the
level-(m-2) children it keeps), its help work once the owner's T(m-1) copy
has landed (copy modelled at RATE_NVLINK after the owner's top level), then
each release group's subtree plan once its sources are done (S5Runner gates
these on CUDA IPC events).  The T(m-2) exchange is fused into the producing
kernels (peer stores over NVLink) and is not modelled.  Printed without and
with helpers.

usage: python tools/s5_timing.py CONFIG [WORLD ...]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs
from paper_1301_7744_b200.distributed import RATE_NVLINK, s5_tasks

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
        for helpers in (False, True):
            replay(m, n, p, ba, bc, w, helpers, A, X, t1, reps)


def replay(m, n, p, ba, bc, w, helpers, A, X, t1, reps):
    """Time every task of the schedule, then replay the job: owner work, the
    T(m-1) peer copy to a helper (modelled at RATE_NVLINK), help work, and
    release groups that start when their sources' events fire."""
    sc = s5_tasks(m, n, p, ba, bc, w, helpers=helpers)
    if helpers and not sc["helper"]:
        return
    owners, subs, groups = sc["owners"], sc["subs"], sc["groups"]
    owner_of = {u: r for r in range(w) for u in owners[r]}
    tops = {}

    def run_plan(pl, inp):
        out = torch.empty(pl.c_elems, dtype=torch.float64, device="cuda")
        t = timed(pl, inp, X, out, reps)
        pl.close()
        return t, out

    own_end, sent, help_end, t_g = [0.0] * w, {}, {}, []
    for r in range(w):
        t = 0.0
        for u in owners[r]:
            if u in sc["helper"]:
                tt, tops[u] = run_plan(bs.SttsmPlan(m, n, p, ba, bc, units=[u], stop_level=m - 1), A)
                sent[u] = tt + tops[u].numel() * 8 / RATE_NVLINK * 1e3
                tl, _ = run_plan(bs.SttsmPlan(m, n, p, ba, bc, start_level=m - 1, start_calls=[(u,)],
                                              start_children=sc["own_children"][u], stop_level=m - 2), tops[u])
                t += tt + tl
        mine = [u for u in owners[r] if u not in sc["helper"]]
        if mine:
            t += run_plan(bs.SttsmPlan(m, n, p, ba, bc, units=mine, stop_level=m - 2), A)[0]
        own_end[r] = t
        torch.cuda.empty_cache()
    for u, (h, kids) in sc["helper"].items():
        th, _ = run_plan(bs.SttsmPlan(m, n, p, ba, bc, start_level=m - 1, start_calls=[(u,)],
                                      start_children=kids, stop_level=m - 2), tops[u])
        help_end[h] = max(own_end[h], sent[u]) + th
    tops.clear()
    torch.cuda.empty_cache()
    for r in range(w):
        tg = []
        for lo, hi, _ in groups[r]:
            pl = bs.SttsmPlan(m, n, p, ba, bc, start_level=m - 2, start_calls=subs[r][lo:hi])
            inp = torch.rand(pl.a_elems, dtype=torch.float64, device="cuda")
            tg.append(round(run_plan(pl, inp)[0], 3))
            del inp
            torch.cuda.empty_cache()
        t_g.append(tg)
    ends = []
    for r in range(w):
        t = max(own_end[r], help_end.get(r, 0.0))
        for (lo, hi, src), tg in zip(groups[r], t_g[r]):
            ready = [own_end[q] if tag == "own" else help_end[q] for q, tag in src]
            t = max([t] + ready) + tg
        ends.append(round(t, 3))
    job = max(ends)
    print(json.dumps({"world": w, "helpers": sc["helper"], "owners": owners,
                      "owner_ms": [round(v, 3) for v in own_end], "help_end_ms": {k: round(v, 3) for k, v in help_end.items()},
                      "groups_ms": t_g, "rank_end_ms": ends, "job_ms_gated": round(job, 3),
                      "eff_gated": round(t1 / w / job, 4), "nvlink_GBps_assumed": RATE_NVLINK / 1e9}), flush=True)


if __name__ == "__main__":
    main()
