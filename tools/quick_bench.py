"""Quick device-resident timing of SttsmPlan on BASELINE configs (dev tool)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs

CFGS = {2: (3, 512, 512, 32, 32), 3: (4, 192, 192, 16, 16), 4: (5, 96, 96, 8, 8), 5: (4, 512, 256, 32, 32)}


def main():
    which = [int(a) for a in sys.argv[1:]] or [2, 3, 4]
    for c in which:
        m, n, p, ba, bc = CFGS[c]
        # QB_PIPELINE=w: a pipelined (mirrored, waved) plan on the device path
        plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=int(os.environ.get("QB_PIPELINE", "0")))
        g = torch.Generator(device="cuda").manual_seed(1)
        A = torch.rand(plan.a_elems, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        X = torch.randn(p, n, dtype=torch.float64, device="cuda", generator=g)
        C = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
        plan.attach_torch_workspace()
        for _ in range(2):
            plan.run(A, X, C)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(5):
            s.record(); plan.run(A, X, C); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
        ms = sorted(ts)[len(ts) // 2]
        fl = plan.stats()["flops"]
        plan.set_timing(True)
        plan.run(A, X, C)
        lv = {}
        for k, f, t in plan.launch_times():
            lv.setdefault(k, [0, 0.0]); lv[k][0] += f; lv[k][1] += t
        plan.set_timing(False)
        print(json.dumps({"config": c, "ms": ms, "tflops": fl / ms / 1e9, "frac_of_37.1": fl / ms / 1e9 / 37.1,
                          "ws_gb": plan.workspace_bytes / 1e9, "launches": plan.last_launches,
                          "levels": {k: [round(v[1], 3), round(v[0] / v[1] / 1e9, 2)] for k, v in lv.items()}}), flush=True)
        del A, X, C, plan
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
