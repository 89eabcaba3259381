"""A/B of libisort builds on u64 keys (keys only; AB_VALS=1: with the position payload): time of the
radix sort of AB_N (default 5e7) seeded 64-bit keys.   python tools/ab_u64.py LIB.so [LIB.so ...]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1206_3511_b200 import _lib

n = int(os.environ.get("AB_N", 50_000_000))
k = np.random.default_rng(3).integers(0, 1 << 63, size=n, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
keys = torch.from_numpy(k.view(np.int64)).cuda()
out = torch.empty_like(keys)
vals = os.environ.get("AB_VALS") == "1"
vout = torch.empty(n, dtype=torch.int32, device="cuda") if vals else None
want = np.sort(k)
for so in sys.argv[1:]:
    lib = ctypes.CDLL(os.path.abspath(so))
    for name, (res, args) in _lib.SIGNATURES.items():
        f = getattr(lib, name, None)
        if f is not None:
            f.restype, f.argtypes = res, args
    tb = lib.isort_radix_temp_bytes(n, 8, 1 if vals else 0)
    temp = torch.empty(tb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def run():
        rc = lib.isort_radix_sort_u64(keys.data_ptr(), out.data_ptr(), None, vout.data_ptr() if vals else None, n,
                                      2 if vals else 0, temp.data_ptr(), tb, s)
        assert rc == 0, rc

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        run()
    b.record()
    torch.cuda.synchronize()
    ok = bool(np.array_equal(out.cpu().numpy().view(np.uint64), want))
    print(os.path.basename(os.path.dirname(so)), f"{a.elapsed_time(b) / 10:.4f} ms/sort  {n / (a.elapsed_time(b) / 10) / 1e6:.1f} Gkeys/s  ok={ok}",
          flush=True)
