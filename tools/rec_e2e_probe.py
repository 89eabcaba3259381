"""Probe: records e2e (radix_sort_lsd on 1e8 host Records) and host memcpy bandwidth;
run with ISORT_STAGING_THREADS=... to compare staging worker counts."""
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
# host memcpy bandwidth, 1 thread
a = np.empty(400_000_000, dtype=np.uint8); b = np.empty_like(a); a[:] = 1; b[:] = 0
t0 = time.perf_counter(); b[:] = a; t = time.perf_counter() - t0
print("numpy 400MB copy GB/s (1 thread):", round(0.4 / t, 1), "nproc", os.cpu_count())
