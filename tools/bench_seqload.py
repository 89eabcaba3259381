"""Throughput of the ISRT loader: file in the page cache -> device keys.

    python tools/bench_seqload.py [n]

Prints one JSON line: our isort_sequence_load (u32 keys, on-device range check)
and the reference's read_sequence_file (oracle/_ref, one host thread) on the
same file, in GB/s of file bytes."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1206_3511_b200 import inputs
from paper_1206_3511_b200 import sequence as sq

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
path = os.path.join(tempfile.gettempdir(), f"isort_bench_{n}.isrt")
keys = inputs.uniform_u32(n).astype(np.uint64)
sq.write_sequence(path, sq.SequenceHeader(1, 0, (1 << 32) - 1, 42), keys)
size = os.path.getsize(path)
with open(path, "rb") as f:  # page cache
    while f.read(1 << 26):
        pass
torch.cuda.init()
hdr, d = sq.load(path, 4)  # warm-up (staging allocation)
times = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hdr, d = sq.load(path, 4)
    torch.cuda.synchronize()
    times.append(time.perf_counter() - t0)
ok = bool(np.array_equal(d.cpu().numpy().view(np.uint32), keys.astype(np.uint32)))
ours = size / min(times) / 1e9
line = {"metric": "ISRT load GB/s (file in page cache -> device keys, range-checked)", "n": n,
        "file_bytes": size, "ours_gbs": ours, "ours_s": min(times), "exact": ok}
try:
    from oracle.binding import Reference

    if Reference.available():
        ref = Reference()
        m = min(n, 20_000_000)
        p2 = path + ".ref"
        sq.write_sequence(p2, sq.SequenceHeader(1, 0, (1 << 32) - 1, 42), keys[:m])
        ref.read_sequence_file(p2, capacity=m)
        t0 = time.perf_counter()
        ref.read_sequence_file(p2, capacity=m)
        dt = time.perf_counter() - t0
        line["reference_gbs"] = os.path.getsize(p2) / dt / 1e9
        line["reference_sample_keys"] = m
        os.remove(p2)
except Exception as e:  # noqa: BLE001
    line["reference_error"] = str(e)
os.remove(path)
print(json.dumps(line))
