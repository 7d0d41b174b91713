"""Device time of reuse=False (plain algorithm-by-blocks) vs reuse=True."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs
from paper_1301_7744_b200.generate import random_bcss_device, random_matrix_device
for cfg in [(3, 512, 512, 32, 32), (4, 192, 192, 16, 16)]:
    m, n, p, ba, bc = cfg
    a = random_bcss_device(m, n, ba, 1); x = random_matrix_device(p, n, 2)
    for reuse in (True, False):
        plan = bs.SttsmPlan(*cfg, reuse=reuse)
        c = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
        plan.run(a, x, c); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(3):
            plan.run(a, x, c)
        e.record(); e.synchronize()
        ms = s.elapsed_time(e) / 3
        fl = bs.bcss_flops(*cfg, reuse=reuse)
        print(cfg, "reuse" if reuse else "no-reuse", round(ms, 3), "ms", round(fl / ms / 1e9, 2), "TF (own flops)")
        plan.close(); del c
