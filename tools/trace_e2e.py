"""Time the pipelined host path (run_host) for config $CFG (default 2) at several wave counts."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs
from paper_1301_7744_b200.generate import random_bcss_device, random_matrix_device

import os
CFGS = {2: (3, 512, 512, 32, 32), 3: (4, 192, 192, 16, 16), 4: (5, 96, 96, 8, 8), 5: (4, 512, 256, 32, 32)}
cfg = CFGS[int(os.environ.get("CFG", "2"))]
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
