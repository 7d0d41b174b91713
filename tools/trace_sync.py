"""Host-polled timeline of one synchronous pipelined host run (dev tool):
BCSS_TRACE=1 python tools/trace_sync.py CONFIG SYM(0|1)."""
import sys, torch
sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs
from paper_1301_7744_b200 import generate
CFGS = {2: (3, 512, 512, 32, 32), 3: (4, 192, 192, 16, 16), 4: (5, 96, 96, 8, 8), 5: (4, 512, 256, 32, 32)}
m, n, p, ba, bc = CFGS[int(sys.argv[1])]
a = generate.random_bcss_device(m, n, ba, 1)
ah = torch.empty(a.numel(), dtype=torch.float64).pin_memory(); ah.copy_(a); del a; torch.cuda.empty_cache()
xh = torch.randn(p, n, dtype=torch.float64).pin_memory()
plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=4, symmetric_upload=sys.argv[2] == "1")
ch = torch.empty(plan.c_elems, dtype=torch.float64).pin_memory()
plan.run_host(ah.numpy(), xh.numpy(), ch.numpy())
import os; os.environ["BCSS_TRACE"] = "1"
plan.run_host(ah.numpy(), xh.numpy(), ch.numpy())
