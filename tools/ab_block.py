"""A/B one-sweep builds: time the radix sort of 1e8 seeded u32 keys with each given libisort build."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1206_3511_b200 import _lib, inputs

n = 100_000_000
keys = torch.from_numpy(inputs.uniform_u32(n).view(np.int32)).cuda()
out = torch.empty_like(keys)
for so in sys.argv[1:]:
    lib = ctypes.CDLL(os.path.abspath(so))
    for name, (res, args) in _lib.SIGNATURES.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    tb = lib.isort_radix_temp_bytes(n, 4, 0)
    temp = torch.empty(tb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        lib.isort_radix_sort_u32(keys.data_ptr(), out.data_ptr(), None, None, n, 0, temp.data_ptr(), tb, s)
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(10):
        lib.isort_radix_sort_u32(keys.data_ptr(), out.data_ptr(), None, None, n, 0, temp.data_ptr(), tb, s)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    o = out.cpu().numpy().view(np.uint32)
    print(f"{os.path.basename(so)}: {ms:.3f} ms  {n / ms / 1e6:.1f} Gkeys/s  sorted={bool(np.all(o[:-1] <= o[1:]))}")
