"""A/B bucket-sort builds: time the bucket sort of 1e8 seeded u32 keys (M = 2^32-1) with each libisort build."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1206_3511_b200 import _lib, inputs

n = int(os.environ.get("AB_N", 100_000_000))
cfg = os.environ.get("AB_CONFIG", "c2")
keys = torch.from_numpy(inputs.config_keys(cfg, n).view(np.int32)).cuda()
bound = inputs.config_range_bound(cfg)
out = torch.empty_like(keys)
ref = None
for so in sys.argv[1:]:
    lib = ctypes.CDLL(os.path.abspath(so))
    for name, (res, args) in _lib.SIGNATURES.items():
        if not hasattr(lib, name):  # older builds: entry points added since
            continue
        f = getattr(lib, name, None)  # older builds lack newer entry points
        if f is None:
            continue
        f.restype, f.argtypes = res, args
    tb = lib.isort_bucket_temp_bytes(n, 4, 0)
    temp = torch.empty(tb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    call = lambda: lib.isort_bucket_sort_u32(keys.data_ptr(), out.data_ptr(), None, None, n, bound, 0,
                                             temp.data_ptr(), tb, s)
    for _ in range(3):
        assert call() == 0
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(10):
        call()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    o = out.cpu().numpy().view(np.uint32)
    if ref is None:
        ref = np.sort(keys.cpu().numpy().view(np.uint32))
    print(f"{os.path.basename(so)}: {ms:.3f} ms  {n / ms / 1e6:.1f} Gkeys/s  exact={bool(np.array_equal(o, ref))}")
