"""Run one BASELINE config's device path twice (dev tool for ncu captures:
skip the first run's launches with --launch-skip)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs

CFGS = {2: (3, 512, 512, 32, 32), 3: (4, 192, 192, 16, 16), 4: (5, 96, 96, 8, 8), 5: (4, 512, 256, 32, 32)}
m, n, p, ba, bc = CFGS[int(sys.argv[1])]
plan = bs.SttsmPlan(m, n, p, ba, bc)
A = torch.rand(plan.a_elems, dtype=torch.float64, device="cuda")
X = torch.randn(p, n, dtype=torch.float64, device="cuda")
C = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
plan.attach_torch_workspace()
for _ in range(2):
    plan.run(A, X, C)
torch.cuda.synchronize()
print("launches per run", plan.last_launches)
