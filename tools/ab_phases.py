"""A/B of libisort builds by phase: per-kernel CUDA-event times (isort_profile_*)
of the radix sort (AB_ALG=bucket: the bucket sort) of 1e8 seeded u32 keys,
averaged over reps.
    python tools/ab_phases.py LIB.so [LIB.so ...]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1206_3511_b200 import _lib, inputs

n = int(os.environ.get("AB_N", 100_000_000))
reps = int(os.environ.get("AB_REPS", 20))
keys = torch.from_numpy(inputs.uniform_u32(n).view(np.int32)).cuda()
out = torch.empty_like(keys)
for so in sys.argv[1:]:
    lib = ctypes.CDLL(os.path.abspath(so))
    for name, (res, args) in _lib.SIGNATURES.items():
        f = getattr(lib, name, None)
        if f is not None:
            f.restype, f.argtypes = res, args
    bucket = os.environ.get("AB_ALG") == "bucket"
    tb = (lib.isort_bucket_temp_bytes if bucket else lib.isort_radix_temp_bytes)(n, 4, 0)
    temp = torch.empty(tb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def run():
        if bucket:
            lib.isort_bucket_sort_u32(keys.data_ptr(), out.data_ptr(), None, None, n, (1 << 32) - 1, 0,
                                      temp.data_ptr(), tb, s)
        else:
            lib.isort_radix_sort_u32(keys.data_ptr(), out.data_ptr(), None, None, n, 0, temp.data_ptr(), tb, s)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    lib.isort_profile_begin()
    for _ in range(reps):
        run()
    torch.cuda.synchronize()
    ms = (ctypes.c_float * 4096)()
    names = ctypes.create_string_buffer(4096 * 16)
    cnt, na = ctypes.c_int(0), ctypes.c_int(0)
    lib.isort_profile_end(ms, names, 16, 4096, ctypes.byref(cnt), ctypes.byref(na))
    acc = {}
    for i in range(cnt.value):
        k = names.raw[i * 16:(i + 1) * 16].split(b"\0")[0].decode()
        acc.setdefault(k, []).append(ms[i])
    ok = bool((out[1:].view(torch.int64 if False else torch.int32).cpu().numpy().view(np.uint32) >=
               out[:-1].cpu().numpy().view(np.uint32)).all())
    print(os.path.basename(os.path.dirname(so)) or so, "sorted" if ok else "NOT SORTED",
          " ".join(f"{k}={np.mean(v):.4f}" for k, v in acc.items()))
