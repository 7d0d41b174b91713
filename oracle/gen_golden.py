"""Generate golden vectors for the BCSS sttsm path by running the REFERENCE.

Run in the build container only (it imports the read-only reference package
from /root/reference/pkg/src; that path does not exist on the GPU box):

    python oracle/gen_golden.py

Writes small ``.npz`` fixtures to ``tests/golden/``.  Every array in them is an
output (or seeded input) of the reference's own public API:
``compress``/``random_symmetric``/``random_matrix``/``random_bcss`` for inputs,
``sttsm_bcss`` (change_of_basis.py:239-284) and ``sttsm_naive``
(change_of_basis.py:77-110) for outputs, ``OpCounter`` flops, ``bcss_costs``
(costs.py:83-142), ``canonicalize`` (indexing.py:34-54),
``hypertriangle_iter`` (indexing.py:57-61), ``save_bcss`` (io.py:50-56).
"""

from __future__ import annotations

import itertools
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import blocksym as ref  # noqa: E402
from blocksym.generate import random_bcss  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
SEED = 20261019


def packed(t) -> np.ndarray:
    """Packed payload of a reference PartialSymTensor/BcssTensor (io.py:53-55)."""
    return np.concatenate([
        np.asarray(t.blocks[key]).reshape(-1, order="F")
        for key in ref.hypertriangle_iter(t.grid, t.sym_modes)
    ]) if t.blocks else np.zeros(0)


def case(name, a_bcss, x, b_c, dense_a=None, store: dict | None = None):
    m, n, b_a = a_bcss.order, a_bcss.n, a_bcss.b
    p = x.shape[0]
    ctr_t, ctr_f = ref.OpCounter(), ref.OpCounter()
    c_true = ref.sttsm_bcss(a_bcss, x, b_c, ctr_t, reuse=True)
    c_false = ref.sttsm_bcss(a_bcss, x, b_c, ctr_f, reuse=False)
    entry = {
        "dims": np.array([m, n, p, b_a, b_c], dtype=np.int64),
        "A": packed(a_bcss),
        "X": np.ascontiguousarray(x, dtype=np.float64),
        "C": packed(c_true),
        "C_noreuse": packed(c_false),
        "flops": np.array([ctr_t.flops, ctr_f.flops], dtype=np.int64),
        "memops": np.array([ctr_t.memops, ctr_f.memops], dtype=np.int64),
    }
    if dense_a is not None:
        naive = ref.sttsm_naive(dense_a, x)
        entry["C_naive"] = packed(ref.compress(naive, b_c, tol=1e-12))
    store[name] = entry


def main() -> None:
    OUT.mkdir(parents=True, exist_ok=True)
    cases: dict = {}

    # BASELINE config 1: symmetrized U(-1,1) dense tensor, X ~ N(0,1).
    a0 = np.random.default_rng(SEED).uniform(-1.0, 1.0, (16,) * 3)
    a_sym = ref.symmetrize(ref.DenseTensor(a0))
    x1 = np.random.default_rng(SEED + 1).standard_normal((16, 16))
    case("config1", ref.compress(a_sym, 4, tol=1e-14), x1, 4, dense_a=a_sym, store=cases)

    # Reference-test shapes (tests/test_change_of_basis.py:113-231): bitwise
    # symmetric inputs via random_symmetric + compress, X ~ U(-1,1).
    small = [
        (2, 4, 4, 1, 1), (2, 4, 4, 2, 2), (2, 8, 8, 2, 2), (3, 4, 4, 2, 2),
        (3, 4, 4, 4, 4), (3, 6, 4, 3, 2), (3, 8, 8, 4, 4), (3, 6, 6, 3, 3),
        (4, 4, 4, 2, 2), (4, 4, 4, 2, 1), (4, 6, 6, 2, 2), (4, 8, 8, 4, 4),
        (5, 4, 4, 2, 2), (5, 6, 6, 3, 3), (5, 8, 8, 4, 4), (3, 8, 12, 2, 4),
        (4, 8, 4, 4, 2), (2, 6, 9, 3, 3), (3, 5, 5, 1, 1),
        # fast-path edge cases: b_C != b_A (both ways), b_C in {1, 2}, large b_C, p < n, p > n
        (3, 16, 8, 4, 1), (3, 16, 16, 4, 2), (3, 16, 32, 4, 16), (3, 32, 16, 16, 4),
        (4, 16, 16, 8, 4), (2, 64, 64, 32, 64), (3, 64, 32, 32, 8), (2, 32, 96, 8, 32),
        # higher orders (the reference supports any m >= 2; this build m <= 8)
        (6, 4, 4, 2, 2), (7, 4, 4, 2, 2), (8, 2, 2, 1, 1), (6, 8, 8, 4, 4),
    ]
    for i, (m, n, p, b_a, b_c) in enumerate(small):
        a = ref.random_symmetric(m, n, SEED + 100 + i)
        x = ref.random_matrix(p, n, SEED + 200 + i)
        case(f"small_m{m}_n{n}_p{p}_ba{b_a}_bc{b_c}", ref.compress(a, b_a), x, b_c,
             dense_a=a, store=cases)

    # random_bcss inputs (generate.py:53-77) with N(0,1) X, as in BASELINE configs 2-5.
    for i, (m, n, b) in enumerate([(3, 16, 4), (4, 12, 4), (5, 8, 2), (3, 32, 8)]):
        a = random_bcss(m, n, b, SEED + 300 + i)
        x = np.random.default_rng(SEED + 301 + i).standard_normal((n, n))
        case(f"rbcss_m{m}_n{n}_b{b}", a, x, b, store=cases)

    for name, entry in cases.items():
        np.savez_compressed(OUT / f"sttsm_{name}.npz", **entry)

    # Temporaries (temp_hook, change_of_basis.py:279-280) in DFS call order.
    a = ref.random_symmetric(4, 4, SEED + 400)
    x = ref.random_matrix(4, 4, SEED + 401)
    seen = []
    ref.sttsm_bcss(ref.compress(a, 2), x, 2, temp_hook=lambda k, t: seen.append((k, packed(t))))
    np.savez_compressed(
        OUT / "temps_m4_n4_b2.npz", A=packed(ref.compress(a, 2)), X=x,
        levels=np.array([k for k, _ in seen], dtype=np.int64),
        **{f"T{i}": t for i, (_, t) in enumerate(seen)})

    # Combinatorics: canonicalize mappings over a full grid, hypertriangle lists.
    idx = list(itertools.product(range(3), repeat=4))
    canon = [ref.canonicalize(i) for i in idx]
    ht = {f"ht_{g}_{m}": np.array(list(ref.hypertriangle_iter(g, m)), dtype=np.int64)
          for g, m in [(1, 3), (3, 3), (5, 2), (4, 4), (16, 3), (12, 5), (6, 1)]}
    np.savez_compressed(
        OUT / "indexing.npz",
        grid_idx=np.array(idx, dtype=np.int64),
        canonical=np.array([c.canonical for c in canon], dtype=np.int64),
        mapping=np.array([c.applied.mapping for c in canon], dtype=np.int64),
        **ht)

    # Cost model (the metric's flop count) for the five BASELINE configs.
    cfgs = [(3, 16, 16, 4, 4), (3, 512, 512, 32, 32), (4, 192, 192, 16, 16),
            (5, 96, 96, 8, 8), (4, 512, 256, 32, 32), (3, 6, 4, 3, 2), (2, 4, 4, 1, 1)]
    rows = []
    for cfg in cfgs:
        for reuse in (True, False):
            rep = ref.bcss_costs(*cfg, meta_k=0, reuse=reuse)
            rows.append(list(cfg) + [int(reuse), rep.flops, rep.memops])
    np.savez_compressed(OUT / "costs.npz", rows=np.array(rows, dtype=np.int64))

    # BCSS file bytes (io.py:50-56) for a small tensor: the packed-buffer contract.
    t = ref.compress(ref.random_symmetric(3, 6, SEED + 500), 2)
    path = OUT / "_tmp.bcss"
    ref.save_bcss(t, path)
    raw = path.read_bytes()
    path.unlink()
    np.savez_compressed(OUT / "bcss_file.npz", raw=np.frombuffer(raw, dtype=np.uint8),
                        A=packed(t), dims=np.array([3, 6, 2], dtype=np.int64))
    print(f"wrote {len(cases) + 4} fixtures to {OUT}")


if __name__ == "__main__":
    main()
