"""Tile-cost calibration on real lower levels (dev tool; feeds csrc/shape_costs.hpp).

For each fast shape (forced with BCSS_FORCE_SHAPE) and each parent height
M = 8 (J+1), run a plan that starts below calls (J, j) of level m-2 (start
calls) and time level m-3, whose parents then all have M rows.  Prints the
device time per parent-row-block so the plan's shape policy can price a tile
holding any number of valid 8-row fragments:
    cost[ba][shape][nf-1] = ms per (call, key, n-tile) of a tile with nf fragments.
"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs

SHAPES_BM = [128, 64, 32, 128, 64, 32, 16, 64, 96, 48]
SHAPES_BN = [128, 256, 256, 128, 256, 256, 512, 256, 128, 256]
CASES = {8: (5, 96, 128), 16: (5, 128, 128), 32: (5, 256, 128)}  # b_a -> (m, n, p); b_c = 8


def level_ms(m, n, p, ba, bc, calls):
    k0 = m - 2
    plan = bs.SttsmPlan(m, n, p, ba, bc, start_level=k0, start_calls=calls)
    g = torch.Generator(device="cuda").manual_seed(1)
    T = torch.rand(plan.a_elems, dtype=torch.float64, device="cuda", generator=g)
    X = torch.randn(p, n, dtype=torch.float64, device="cuda", generator=g)
    C = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
    plan.attach_torch_workspace()
    plan.set_timing(True)
    best = None
    for _ in range(4):
        plan.run(T, X, C)
        torch.cuda.synchronize()
        t = sum(ms for k, _, ms in plan.launch_times() if k == k0 - 1)
        best = t if best is None else min(best, t)
    plan.close()
    del T, X, C
    return best


def one(ba, shape):
    """Fragment costs of one shape (own process: the plan reads BCSS_FORCE_SHAPE once)."""
    m, n, p = CASES[ba]
    pbar = p // 8
    from math import comb
    keys = comb(n // ba + (m - 3) - 1, m - 3)
    rest = ba ** (m - 3) * 8 ** 2
    bm = SHAPES_BM[shape]
    ntiles = -(-rest // SHAPES_BN[shape])
    costs = []
    for nf in range(1, bm // 8 + 1):
        J = nf - 1
        calls = [(J, j) for j in range(J, min(pbar, J + 4))]
        costs.append(level_ms(m, n, p, ba, 8, calls) / (len(calls) * keys * ntiles))
    tf = 2 * bm * n * SHAPES_BN[shape] / (costs[-1] * 1e-3) / 1e12
    print(json.dumps({"ba": ba, "shape": shape, "full_tile_tflops": round(tf, 2),
                      "frac": [round(c / costs[-1], 4) for c in costs]}), flush=True)


def main():
    if len(sys.argv) == 4 and sys.argv[1] == "--one":
        return one(int(sys.argv[2]), int(sys.argv[3]))
    import subprocess
    bas = [int(a) for a in sys.argv[1:]] or [8, 16, 32]
    out = {}
    for ba in bas:
        rows = []
        for shape in range(len(SHAPES_BM)):
            env = dict(os.environ, BCSS_FORCE_SHAPE=str(shape))
            res = subprocess.run([sys.executable, __file__, "--one", str(ba), str(shape)], env=env,
                                 capture_output=True, text=True)
            line = [l for l in res.stdout.splitlines() if l.startswith("{")][-1]
            print(line, flush=True)
            rows.append(json.loads(line))
        out[ba] = {"full_tflops": [r["full_tile_tflops"] for r in rows], "frac": [r["frac"] for r in rows]}
    print(json.dumps(out))


def _unused():
    bas = []
    out = {}
    for ba in bas:
        m, n, p = CASES[ba]
        pbar = p // 8
        nbar = n // ba
        from math import comb
        keys = comb(nbar + (m - 3) - 1, m - 3)
        rest = ba ** (m - 3) * 8 ** 2
        per_shape = []
        for shape, bm in enumerate(SHAPES_BM):
            os.environ["BCSS_FORCE_SHAPE"] = str(shape)
            ntiles = -(-rest // SHAPES_BN[shape])
            costs = []
            for nf in range(1, bm // 8 + 1):
                J = nf - 1
                calls = [(J, j) for j in range(J, min(pbar, J + 4))]
                ms = level_ms(m, n, p, ba, 8, calls)
                costs.append(ms / (len(calls) * keys * ntiles))
                if os.environ.get("CAL_DEBUG"):
                    print("  nf", nf, "calls", len(calls), "ms", round(ms, 4), flush=True)
            full = costs[-1]
            per_shape.append([round(c / full, 4) for c in costs])
            tf = 2 * bm * n * SHAPES_BN[shape] / (full * 1e-3) / 1e12
            print(json.dumps({"ba": ba, "shape": shape, "full_tile_tflops": round(tf, 2),
                              "frac": per_shape[-1]}), flush=True)
        out[ba] = per_shape
        torch.cuda.empty_cache()
    os.environ.pop("BCSS_FORCE_SHAPE", None)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
