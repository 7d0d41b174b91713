"""Measure each fast tile shape's full-tile FP64 throughput per b_a (feeds
ShapePolicy::eff in csrc/bcss_capi.cu).  Runs the top level of configs 2/3/4
(one parent with rows = p) with BCSS_FORCE_SHAPE and corrects for padding."""
import json
import math
import os
import subprocess
import sys

SHAPES_BM = [128, 64, 32, 128, 64, 32, 16, 64, 96, 48]
CASES = {32: (2, 512), 16: (3, 192), 8: (4, 96)}  # b_a -> (config, rows at top level)
out = {}
for shape, bm in enumerate(SHAPES_BM):
    env = dict(os.environ, BCSS_FORCE_SHAPE=str(shape))
    res = subprocess.run([sys.executable, "tools/quick_bench.py", "2", "3", "4"], env=env,
                         capture_output=True, text=True)
    lines = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    for ba, (cfg, rows) in CASES.items():
        d = next(l for l in lines if l["config"] == cfg)
        top = max(d["levels"], key=int)
        pad = rows / (math.ceil(rows / bm) * bm)
        out.setdefault(ba, [0.0] * len(SHAPES_BM))[shape] = round(d["levels"][top][1] / pad, 2)
print(json.dumps(out))
