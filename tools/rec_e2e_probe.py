"""Probe: records e2e (radix_sort_lsd on 1e8 host Records), pinned H2D/D2H of the
same size, host memcpy bandwidth, and the call into a reused (faulted-in) output.
Run with ISORT_HOST_TRACE=1 for the upload / sort / download split and with
ISORT_STAGING_THREADS=... to compare staging worker counts."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1206_3511_b200 as isort
from paper_1206_3511_b200 import inputs
from paper_1206_3511_b200.intsort import RECORD_DTYPE
n = 100_000_000
seq = np.empty(n, dtype=RECORD_DTYPE)
seq["key"] = inputs.config_keys("c2", n)
seq["tag"] = np.arange(n, dtype=np.uint64)
out = isort.radix_sort_lsd(seq, 256)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); out = isort.radix_sort_lsd(seq, 256); ts.append(time.perf_counter() - t0)
print(os.environ.get("ISORT_STAGING_THREADS"), "records e2e ms:", [round(t * 1e3, 1) for t in ts])
# host memcpy bandwidth, 1 thread; pinned H2D / D2H of the records' size
import torch
h = torch.empty(16 * n, dtype=torch.uint8).pin_memory(); d = torch.empty(16 * n, dtype=torch.uint8, device="cuda")
for _ in range(2):
    t0 = time.perf_counter(); d.copy_(h); torch.cuda.synchronize(); t1 = time.perf_counter(); h.copy_(d); torch.cuda.synchronize(); t2 = time.perf_counter()
print("pinned 1.6 GB H2D %.1f ms, D2H %.1f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3))
del h, d
a = np.empty(400_000_000, dtype=np.uint8); b = np.empty_like(a); a[:] = 1; b[:] = 0
t0 = time.perf_counter(); b[:] = a; t = time.perf_counter() - t0
print("numpy 400MB copy GB/s (1 thread):", round(0.4 / t, 1), "nproc", os.cpu_count())
# the same call into a reused (already faulted-in) output buffer
from paper_1206_3511_b200 import _lib
lib = _lib.load()
out2 = np.empty_like(seq)
out2["key"] = 0
for _ in range(3):
    t0 = time.perf_counter()
    _lib.check(lib.isort_radix_sort_records(seq.ctypes.data, out2.ctypes.data, n, 256, 0))
    print("reused output buffer: %.1f ms" % ((time.perf_counter() - t0) * 1e3))
