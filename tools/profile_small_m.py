"""One level with single-m-tile parents (dev tool for ncu): start below calls
(J, j) of level m-2 with a forced shape; the first level kernel launched is
level m-3 whose parents all have 8 (J+1) rows."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs

shape = int(sys.argv[1]) if len(sys.argv) > 1 else 2
J = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ba = int(sys.argv[3]) if len(sys.argv) > 3 else 8
os.environ["BCSS_FORCE_SHAPE"] = str(shape)
m, n, p = {8: (5, 96, 128), 16: (5, 128, 128), 32: (5, 256, 128)}[ba]
calls = [(J, j) for j in range(J, min(p // 8, J + 4))]
plan = bs.SttsmPlan(m, n, p, ba, 8, start_level=m - 2, start_calls=calls)
T = torch.rand(plan.a_elems, dtype=torch.float64, device="cuda")
X = torch.randn(p, n, dtype=torch.float64, device="cuda")
C = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
plan.attach_torch_workspace()
for _ in range(2):
    plan.run(T, X, C)
torch.cuda.synchronize()
print("ok")
