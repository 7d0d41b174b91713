"""Repeat every golden case several times through the drop-in; report mismatches."""
import glob
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs
from oracle import bcss_oracle as orc

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
pat = sys.argv[2] if len(sys.argv) > 2 else "*"
bad = 0
for path in sorted(glob.glob(f"tests/golden/sttsm_{pat}.npz")):
    d = np.load(path)
    m, n, p, ba, bc = (int(v) for v in d["dims"])
    for reuse in (True, False):
        want = d["C"] if reuse else d["C_noreuse"]
        for r in range(reps):
            out = bs.sttsm_bcss(bs.BcssTensor(m, n, ba, payload=d["A"]), d["X"], bc, reuse=reuse)
            err = orc.rel_frobenius(out.payload, want)
            if not err <= 1e-12:
                bad += 1
                diff = np.abs(out.payload - want).reshape(-1, bc**m).max(axis=1)
                print(f"MISMATCH {path.split('/')[-1]} reuse={reuse} rep={r} err={err:.3e} "
                      f"bad_blocks={np.nonzero(diff > 1e-10 * np.abs(want).max())[0].tolist()[:10]}")
print(f"done, {bad} mismatches")
