"""D2H of many block-sized copies over 1..8 streams, and SM stores into mapped
pinned host memory (dev tool: e2e download design)."""
import json
import time

import torch

n = 216 * 1024 * 1024 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.randn(n, dtype=torch.float64, device="cuda")


def timeit(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


out = {}
for chunk in (256 << 10, 1 << 20):
    k = chunk // 8
    for ns in (1, 2, 4, 8):
        streams = [torch.cuda.Stream() for _ in range(ns)]

        def many():
            for i, off in enumerate(range(0, n - k + 1, k)):
                with torch.cuda.stream(streams[i % ns]):
                    h[off:off + k].copy_(d[off:off + k], non_blocking=True)
        t = timeit(many)
        out[f"{chunk >> 10}KB_x{ns}streams_GBps"] = round(n * 8 / 1e9 / t, 1)
# SM stores into host memory (torch copy kernel from device to a host-mapped view is not
# exposed; use a strided gather via index_select into a pinned-mapped tensor is also not
# possible) -> measured with the library's probe when present
print(json.dumps(out))
