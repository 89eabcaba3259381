"""Per-phase cycle split of the one-sweep pass (debug build with -DISORT_PHASE_TIMING).

Builds tools/libisort_timing.so, sorts 1e8 keys once per digit slot, and reads the
accumulated clock64 deltas that the instrumented kernel leaves in RadixState.hist
(the histograms are no longer needed when a pass runs)."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
so = os.path.join(ROOT, "tools", "libisort_timing.so")
if not os.path.exists(so) or "--rebuild" in sys.argv:
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                    "-DISORT_PHASE_TIMING", "-Xcompiler", "-fPIC", "-shared", "-o", so,
                    os.path.join(ROOT, "paper_1206_3511_b200", "csrc", "isort_api.cu")], check=True)
if "--build-only" in sys.argv:
    sys.exit(0)
import numpy as np
import torch

from paper_1206_3511_b200 import _lib, inputs

lib = ctypes.CDLL(so)
for name, (res, args) in _lib.SIGNATURES.items():
    f = getattr(lib, name)
    f.restype, f.argtypes = res, args
n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 100_000_000
keys = torch.from_numpy(inputs.uniform_u32(n).view(np.int32)).cuda()
out = torch.empty_like(keys)
tb = lib.isort_radix_temp_bytes(n, 4, 0)
temp = torch.empty(tb, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for rep in range(1):
    assert lib.isort_radix_sort_u32(keys.data_ptr(), out.data_ptr(), None, None, n, 0, temp.data_ptr(), tb, s) == 0
    torch.cuda.synchronize()
# RadixState at offset 0 of temp; offs[7][0..7] (unused for u32 keys) holds 4 u64 accumulators
off = 4 * (8 * 256) + 4 * (7 * 256)  # RadixState.offs[7][0]
acc = temp[off:off + 48].cpu().numpy().view(np.uint64)
tiles = int(acc[3])
print(f"tiles={tiles}  cycles/tile: phase1={acc[0] / tiles:.0f}  serial={acc[1] / tiles:.0f}  phase2={acc[2] / tiles:.0f}"
      f"  [serial: pre-lookback={acc[4] / tiles:.0f} lookback={acc[5] / tiles:.0f}]")
