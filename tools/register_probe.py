"""Cost of cudaHostRegister on pageable numpy buffers vs pageable copies (dev tool)."""
import ctypes
import json
import time

import numpy as np
import torch

cudart = ctypes.CDLL("libcudart.so")
n = 216 * 1024 * 1024 // 8
h = np.random.default_rng(0).standard_normal(n)
d = torch.empty(n, dtype=torch.float64, device="cuda")
out = {}
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    d.copy_(torch.from_numpy(h))
    torch.cuda.synchronize()
    out[f"pageable_h2d_ms_{rep}"] = round((time.perf_counter() - t0) * 1e3, 3)
    t0 = time.perf_counter()
    r = cudart.cudaHostRegister(ctypes.c_void_p(h.ctypes.data), ctypes.c_size_t(h.nbytes), 0)
    t1 = time.perf_counter()
    d.copy_(torch.from_numpy(h), non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cudart.cudaHostUnregister(ctypes.c_void_p(h.ctypes.data))
    t3 = time.perf_counter()
    out[f"register_ms_{rep}"] = round((t1 - t0) * 1e3, 3)
    out[f"registered_h2d_ms_{rep}"] = round((t2 - t1) * 1e3, 3)
    out[f"unregister_ms_{rep}"] = round((t3 - t2) * 1e3, 3)
    out["register_status"] = r
print(json.dumps(out))
