"""A/B one-sweep builds: time the radix sort of 1e8 seeded u32 keys with each given libisort build."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1206_3511_b200 import _lib, inputs

n = int(os.environ.get("AB_N", 100_000_000))
mode = int(os.environ.get("AB_VALS", "0"))  # 0 keys only, 2 iota payload
k64 = os.environ.get("AB_KEY64") == "1"
if k64:
    hk = inputs.uniform_u32(n).astype(np.uint64) << np.uint64(32) | inputs.uniform_u32(n, seed=7).astype(np.uint64)
    keys = torch.from_numpy(hk.view(np.int64)).cuda()
else:
    keys = torch.from_numpy(inputs.uniform_u32(n).view(np.int32)).cuda()
out = torch.empty_like(keys)
vout = torch.empty(n, dtype=torch.int32, device="cuda") if mode else None
for so in sys.argv[1:]:
    lib = ctypes.CDLL(os.path.abspath(so))
    for name, (res, args) in _lib.SIGNATURES.items():
        f = getattr(lib, name, None)  # older builds lack newer entry points
        if f is None:
            continue
        f.restype, f.argtypes = res, args
    tb = lib.isort_radix_temp_bytes(n, 8 if k64 else 4, mode)
    sortfn = lib.isort_radix_sort_u64 if k64 else lib.isort_radix_sort_u32
    temp = torch.empty(tb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        sortfn(keys.data_ptr(), out.data_ptr(), None, vout.data_ptr() if mode else None, n, mode,
                                 temp.data_ptr(), tb, s)
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(10):
        sortfn(keys.data_ptr(), out.data_ptr(), None, vout.data_ptr() if mode else None, n, mode,
                                 temp.data_ptr(), tb, s)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    o = out.cpu().numpy().view(np.uint64 if k64 else np.uint32)
    print(f"{os.path.basename(so)}: {ms:.3f} ms  {n / ms / 1e6:.1f} Gkeys/s  sorted={bool(np.all(o[:-1] <= o[1:]))}")
