"""Cost of partial tiles (dev tool): for each fast shape and each count of
valid 8-row fragments, time the top level of a problem whose only parent has
exactly that many rows (one tile per (key, n-tile)), relative to a full tile.
Feeds ShapePolicy's partial-tile model in csrc/plan.cu."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs

SHAPES_BM = [128, 64, 32, 128, 64, 32, 16, 64, 96, 48]
CASES = {8: (5, 96, 8), 16: (5, 128, 16), 32: (4, 256, 32)}  # b_a -> (m, n, b_a); b_c = 8, p = rows


def top_ms(m, n, p, ba, bc):
    plan = bs.SttsmPlan(m, n, p, ba, bc, stop_level=m - 1)
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.rand(plan.a_elems, dtype=torch.float64, device="cuda", generator=g)
    X = torch.randn(p, n, dtype=torch.float64, device="cuda", generator=g)
    C = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
    plan.attach_torch_workspace()
    plan.run(A, X, C)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        s.record(); plan.run(A, X, C); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    ms = sorted(ts)[2]
    fl = plan.stats()["flops"]
    plan.close()
    del A, X, C
    return ms, fl


def main():
    bas = [int(a) for a in sys.argv[1:]] or [8, 16, 32]
    out = {}
    for ba in bas:
        m, n, _ = CASES[ba]
        rows = {}
        for shape, bm in enumerate(SHAPES_BM):
            os.environ["BCSS_FORCE_SHAPE"] = str(shape)
            full_ms, full_fl = top_ms(m, n, bm, ba, 8)
            fr = []
            for v in range(8, bm + 1, 8):
                ms, _ = top_ms(m, n, v, ba, 8) if v < bm else (full_ms, full_fl)
                fr.append(round(ms / full_ms, 4))
            rows[shape] = {"full_tflops": round(full_fl / full_ms / 1e9, 2), "frac": fr}
            print(json.dumps({"ba": ba, "shape": shape, **rows[shape]}), flush=True)
        out[ba] = rows
        torch.cuda.empty_cache()
    os.environ.pop("BCSS_FORCE_SHAPE", None)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
