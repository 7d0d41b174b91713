"""Time the pipelined host path (run_host) for config 2 at several wave counts."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs
from paper_1301_7744_b200.generate import random_bcss_device, random_matrix_device

cfg = (3, 512, 512, 32, 32)
m, n, p, ba, bc = cfg
a = random_bcss_device(m, n, ba, 1).cpu().pin_memory()
x = random_matrix_device(p, n, 2).cpu().pin_memory()
for w in [int(v) for v in sys.argv[1:]] or [4]:
    plan = bs.SttsmPlan(*cfg, pipeline=w)
    c = torch.empty(plan.c_elems, dtype=torch.float64).pin_memory()
    for _ in range(2):
        plan.run_host(a.numpy(), x.numpy(), c.numpy())
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        plan.run_host(a.numpy(), x.numpy(), c.numpy())
        ts.append((time.perf_counter() - t0) * 1e3)
    print(w, "min %.3f median %.3f ms" % (min(ts), sorted(ts)[5]), flush=True)
    plan.close()
