"""Wall time of the drop-in sttsm_bcss (reference call shape, numpy in/out)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs
from oracle import bcss_oracle as orc

for name, (m, n, p, ba, bc) in {"config 1": (3, 16, 16, 4, 4), "config 2": (3, 512, 512, 32, 32)}.items():
    a = bs.BcssTensor(m, n, ba, payload=orc.random_bcss_packed(m, n, ba, 1))
    x = np.random.default_rng(2).standard_normal((p, n))
    ts = []
    for i in range(6):
        t0 = time.perf_counter()
        out = bs.sttsm_bcss(a, x, bc)
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"drop-in sttsm_bcss {name} wall ms:", [round(t, 2) for t in ts])
