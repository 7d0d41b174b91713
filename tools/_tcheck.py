import os, sys, torch
sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import calibrate_level as cl
import paper_1301_7744_b200 as bs
os.environ["BCSS_FORCE_SHAPE"] = "2"
for rep in range(2):
    m, n, p, ba = 5, 96, 128, 8
    calls = [(3, j) for j in range(3, 7)]
    plan = bs.SttsmPlan(m, n, p, ba, 8, start_level=m - 2, start_calls=calls)
    g = torch.Generator(device="cuda").manual_seed(1)
    T = torch.rand(plan.a_elems, dtype=torch.float64, device="cuda", generator=g)
    X = torch.randn(p, n, dtype=torch.float64, device="cuda", generator=g)
    C = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
    plan.attach_torch_workspace()
    plan.set_timing(True)
    for _ in range(4):
        plan.run(T, X, C)
        torch.cuda.synchronize()
        print(plan.launch_times())
    plan.close()
print(cl.level_ms(5, 96, 128, 8, 8, calls))
