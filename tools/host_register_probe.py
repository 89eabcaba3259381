"""Probe: cost of cudaHostRegister / Unregister on a fresh and a touched 1.6 GB
numpy buffer (is pinning the caller's records in place cheaper than staging?)."""
import ctypes
import time

import numpy as np
import torch

cudart = ctypes.CDLL("libcudart.so") if False else None
torch.cuda.init()
rt = torch.cuda.cudart()
n = 1_600_000_000
for label, a in (("touched", np.ones(n, dtype=np.uint8)), ("fresh", np.empty(n, dtype=np.uint8))):
    for _ in range(2):
        t0 = time.perf_counter()
        rc = rt.cudaHostRegister(a.ctypes.data, n, 0)
        t1 = time.perf_counter()
        d = torch.empty(n, dtype=torch.uint8, device="cuda")
        h = torch.from_numpy(a)
        t2 = time.perf_counter()
        d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        rt.cudaHostUnregister(a.ctypes.data)
        t4 = time.perf_counter()
        print(f"{label}: register {1e3 * (t1 - t0):.1f} ms (rc {rc}), H2D {1e3 * (t3 - t2):.1f} ms, "
              f"unregister {1e3 * (t4 - t3):.1f} ms")
