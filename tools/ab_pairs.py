import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1206_3511_b200 import _lib, inputs
n = int(os.environ.get("AB_N", 100_000_000))
keys = torch.from_numpy(inputs.uniform_u32(n).view(np.int32)).cuda()
out = torch.empty_like(keys); vout = torch.empty_like(keys)
for so in sys.argv[1:]:
    lib = ctypes.CDLL(os.path.abspath(so))
    for name, (res, args) in _lib.SIGNATURES.items():
        f = getattr(lib, name, None)
        if f is not None: f.restype, f.argtypes = res, args
    tb = lib.isort_radix_temp_bytes(n, 4, 1)
    temp = torch.empty(tb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    def run():
        rc = lib.isort_radix_sort_u32(keys.data_ptr(), out.data_ptr(), None, vout.data_ptr(), n, 2, temp.data_ptr(), tb, s)
        assert rc == 0, rc
    for _ in range(3): run()
    torch.cuda.synchronize()
    lib.isort_profile_begin()
    for _ in range(10): run()
    torch.cuda.synchronize()
    ms = (ctypes.c_float * 4096)(); names = ctypes.create_string_buffer(4096 * 16)
    cnt, na = ctypes.c_int(0), ctypes.c_int(0)
    lib.isort_profile_end(ms, names, 16, 4096, ctypes.byref(cnt), ctypes.byref(na))
    acc = {}
    for i in range(cnt.value):
        k = names.raw[i * 16:(i + 1) * 16].split(b"\0")[0].decode(); acc.setdefault(k, []).append(ms[i])
    print(os.path.basename(os.path.dirname(so)), " ".join(f"{k}={np.mean(v):.4f}" for k, v in acc.items()), flush=True)
