"""cuBLAS DGEMM (torch.matmul float64) throughput on this GPU: roofline denominator.

Burst = best of 10 at 8192^3; sustained = back-to-back for ~4 s. Prints JSON lines.
"""
import json
import time

import torch


def main():
    dev = torch.device("cuda:0")
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device=dev)
        b = torch.randn(n, n, dtype=torch.float64, device=dev)
        for _ in range(3):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 1e30
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(10):
            s.record(); torch.matmul(a, b); e.record(); e.synchronize()
            best = min(best, s.elapsed_time(e))
        print(json.dumps({"kind": "cublas_dgemm_burst", "n": n, "tflops": 2 * n**3 / best / 1e9}))
    t0 = time.time(); cnt = 0
    s.record()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b); cnt += 1
        if cnt % 8 == 0:
            torch.cuda.synchronize()
    e.record(); e.synchronize()
    print(json.dumps({"kind": "cublas_dgemm_sustained", "n": 8192, "tflops": cnt * 2 * 8192**3 / s.elapsed_time(e) / 1e9}))


if __name__ == "__main__":
    main()
