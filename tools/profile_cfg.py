"""Run one BASELINE config's device path (dev tool for ncu captures).

    python tools/profile_cfg.py CFG [--once]

Twice by default (skip the first run's launches with --launch-skip for a
warm capture); ``--once`` runs it a single time, deterministically (fixed
seeds), for ``ncu --replay-mode application``, which re-runs the whole
process once per metric pass instead of saving and restoring the ~130 GB of
device memory a config-5 level kernel can touch."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs

CFGS = {2: (3, 512, 512, 32, 32), 3: (4, 192, 192, 16, 16), 4: (5, 96, 96, 8, 8), 5: (4, 512, 256, 32, 32)}
m, n, p, ba, bc = CFGS[int(sys.argv[1])]
runs = 1 if "--once" in sys.argv else 2
plan = bs.SttsmPlan(m, n, p, ba, bc)
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.rand(plan.a_elems, dtype=torch.float64, device="cuda", generator=g)
X = torch.randn(p, n, dtype=torch.float64, device="cuda", generator=g)
C = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
plan.attach_torch_workspace()
for _ in range(runs):
    plan.run(A, X, C)
torch.cuda.synchronize()
print("launches per run", plan.last_launches)
