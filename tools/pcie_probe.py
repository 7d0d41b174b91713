"""Host<->device copy rates on this box (pinned memory), alone and concurrent."""
import json
import time

import torch

n = 216 * 1024 * 1024 // 8
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


gb = n * 8 / 1e9
h2d = timeit(lambda: d1.copy_(h1, non_blocking=True))
d2h = timeit(lambda: h2.copy_(d2, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


bi = timeit(both)
print(json.dumps({"bytes_GB": gb, "h2d_GBps": gb / h2d, "d2h_GBps": gb / d2h, "h2d_ms": h2d * 1e3,
                  "d2h_ms": d2h * 1e3, "concurrent_ms": bi * 1e3, "concurrent_GBps_total": 2 * gb / bi}))

# many medium copies (the per-wave C download pattern)
for chunk in (256 << 10, 768 << 10, 4 << 20):
    k = chunk // 8
    s2 = torch.cuda.Stream()

    def many():
        with torch.cuda.stream(s2):
            for off in range(0, n - k + 1, k):
                h2[off:off + k].copy_(d2[off:off + k], non_blocking=True)

    t = timeit(many, reps=3)
    print(json.dumps({"d2h_chunk_bytes": chunk, "copies": n // k, "ms": t * 1e3, "GBps": gb / t}))
