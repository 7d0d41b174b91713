"""Per-level device time of reuse=False plans (dev tool)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs
from paper_1301_7744_b200.generate import random_bcss_device, random_matrix_device
for cfg in [(3, 512, 512, 32, 32), (4, 192, 192, 16, 16), (5, 96, 96, 8, 8)]:
    m, n, p, ba, bc = cfg
    a = random_bcss_device(m, n, ba, 1); x = random_matrix_device(p, n, 2)
    plan = bs.SttsmPlan(*cfg, reuse=False)
    c = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
    plan.run(a, x, c); torch.cuda.synchronize()
    plan.set_timing(True); plan.run(a, x, c); torch.cuda.synchronize()
    lv = {}
    for k, f, t in plan.launch_times():
        lv.setdefault(k, [0, 0.0]); lv[k][0] += f; lv[k][1] += t
    tot = sum(v[1] for v in lv.values())
    print(cfg, "total %.2f ms" % tot, {k: (round(v[1], 2), round(v[0] / v[1] / 1e9, 1)) for k, v in lv.items()}, flush=True)
    plan.close(); del a, x, c; torch.cuda.empty_cache()
