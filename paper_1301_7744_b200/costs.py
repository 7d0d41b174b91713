"""The metric's work count: exact flops of the blocked algorithm.

``bcss_flops`` is ``bcss_costs(m, n, p, b_a, b_c, reuse=...).flops``
(/root/reference/pkg/src/blocksym/costs.py:83-112), evaluated by the native
library in 128-bit integers.  ``bcss_memops`` is the same model's memop count
(costs.py:112), which the drop-in reports to an ``OpCounter`` because the
GPU path folds the reference's explicit permutations into its loads.
"""

from __future__ import annotations

import ctypes
import math
from fractions import Fraction

from . import _native
from .errors import ParameterError


def bcss_flops(m: int, n: int, p: int, b_a: int, b_c: int, reuse: bool = True) -> int:
    out = ctypes.c_uint64()
    _native.check(_native.lib().bcss_blocked_flops(m, n, p, b_a, b_c, int(reuse), ctypes.byref(out)))
    return int(out.value)


def bcss_memops(m: int, n: int, p: int, b_a: int, b_c: int, reuse: bool = True) -> int:
    if m < 2 or min(n, p, b_a, b_c) < 1 or n % b_a or p % b_c:
        raise ParameterError("invalid blocked problem")
    nbar, pbar = n // b_a, p // b_c
    ratio = Fraction(b_c, b_a)

    def blocks_of(d: int) -> int:
        if not reuse:
            return nbar ** (m - 1 - d)
        return math.comb(nbar + m - d - 2, m - d - 1) if m - d - 1 >= 1 else 1

    core = sum(math.comb(pbar + d, d + 1) * blocks_of(d) * ratio**d for d in range(m))
    memops = (nbar + 2 * ratio) * b_a**m * core
    if memops.denominator != 1:
        raise ParameterError("memop count did not reduce to an integer")
    return int(memops)
