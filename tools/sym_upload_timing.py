"""End-to-end host runs with and without the symmetric upload (dev tool).

usage: python tools/sym_upload_timing.py [configs...] [--steps K]
For each BASELINE config: exactly symmetric A (random_bcss_device), pinned
host buffers, a pipelined plan (pipeline=4) with the full upload and one with
the symmetric upload: K streamed calls (run_host_async, consecutive calls
overlapped) and K synchronous calls, CUDA-event timed; C compared bitwise."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1301_7744_b200 as bs
from paper_1301_7744_b200 import generate

CFGS = {2: (3, 512, 512, 32, 32), 3: (4, 192, 192, 16, 16), 4: (5, 96, 96, 8, 8), 5: (4, 512, 256, 32, 32)}


def timed(fn, k):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    fn(k)
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / k


def main():
    argv = sys.argv[1:]
    k = 5
    if "--steps" in argv:
        i = argv.index("--steps")
        k = int(argv[i + 1])
        del argv[i:i + 2]
    which = [int(a) for a in argv] or [2, 3, 4, 5]
    for c in which:
        m, n, p, ba, bc = CFGS[c]
        a_dev = generate.random_bcss_device(m, n, ba, 20261019)
        a_h = torch.empty(a_dev.numel(), dtype=torch.float64).pin_memory()
        a_h.copy_(a_dev)
        del a_dev
        torch.cuda.empty_cache()
        x_h = torch.randn(p, n, dtype=torch.float64, generator=torch.Generator().manual_seed(3)).pin_memory()
        res = {"config": c}
        cs = {}
        for mode in ("full", "sym"):
            plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=4, symmetric_upload=(mode == "sym"))
            c_h = torch.empty(plan.c_elems, dtype=torch.float64).pin_memory()
            A, X, C = a_h.numpy(), x_h.numpy(), c_h.numpy()
            for _ in range(2):
                plan.run_host(A, X, C)

            def stream(kk):
                for _ in range(kk):
                    plan.run_host_async(A, X, C)
                plan.wait()

            def sync(kk):
                for _ in range(kk):
                    plan.run_host(A, X, C)

            stream(2)
            res[mode] = {"streamed_ms": round(timed(stream, k), 3), "sync_ms": round(timed(sync, k), 3),
                         "upload_gb": round(plan.last_upload_bytes / 1e9, 3)}
            cs[mode] = c_h.clone()
            plan.close()
            torch.cuda.empty_cache()
        res["bitwise_equal"] = bool(torch.equal(cs["full"], cs["sym"]))
        res["a_gb"] = round(a_h.numel() * 8 / 1e9, 3)
        print(json.dumps(res), flush=True)
        del a_h, cs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
