"""Device timeline of streamed pipelined host runs (dev tool):
BCSS_TRACE=3 python tools/trace_streamed.py CONFIG SYM(0|1) [K]."""
import sys, os, torch
sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs
from paper_1301_7744_b200 import generate
CFGS = {2: (3, 512, 512, 32, 32), 3: (4, 192, 192, 16, 16), 4: (5, 96, 96, 8, 8), 5: (4, 512, 256, 32, 32)}
m, n, p, ba, bc = CFGS[int(sys.argv[1])]
a = generate.random_bcss_device(m, n, ba, 1)
ah = torch.empty(a.numel(), dtype=torch.float64).pin_memory(); ah.copy_(a); del a; torch.cuda.empty_cache()
xh = torch.randn(p, n, dtype=torch.float64).pin_memory()
plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=int(os.environ.get("PW", "4")), symmetric_upload=sys.argv[2] == "1")
ch = torch.empty(plan.c_elems, dtype=torch.float64).pin_memory()
for _ in range(2):
    plan.run_host_async(ah.numpy(), xh.numpy(), ch.numpy())
plan.wait()
k = int(sys.argv[3]) if len(sys.argv) > 3 else 4
for _ in range(k):
    plan.run_host_async(ah.numpy(), xh.numpy(), ch.numpy())
plan.wait()
