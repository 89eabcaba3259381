"""Per-phase cycle split of the one-sweep pass (debug build with -DISORT_PHASE_TIMING).

Builds tools/libisort_timing.so, sorts 1e8 keys once per digit slot, and reads the
accumulated clock64 deltas that the instrumented kernel leaves in RadixState.hist
(the histograms are no longer needed when a pass runs)."""
import ctypes
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
so = os.path.join(ROOT, "tools", "libisort_timing.so")
libs = [a for a in sys.argv[1:] if a.endswith(".so")]  # a -DISORT_PHASE_TIMING build made by tools/build_variant.py
if libs:
    so = os.path.abspath(libs[0])
elif not os.path.exists(so) or "--rebuild" in sys.argv:
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                    "-DISORT_PHASE_TIMING", "-Xcompiler", "-fPIC", "-shared", "-o", so,
                    *sorted(glob.glob(os.path.join(ROOT, "paper_1206_3511_b200", "csrc", "*.cu")))], check=True)
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
# RadixState (radix_onesweep.cuh) at offset 0 of temp: prof[0..2] accumulate
# phase-1 cycles, phase-2 cycles and tiles over all passes.
import ctypes as C


class RadixState(C.Structure):
    _fields_ = [("hist", C.c_uint32 * 2048), ("offs", C.c_uint32 * 2048), ("max_key", C.c_uint64),
                ("first_bad", C.c_uint64), ("descents", C.c_uint32), ("ascents", C.c_uint32),
                ("n_active", C.c_uint32), ("copy_in_to_out", C.c_uint32), ("reversed", C.c_uint32), ("counting", C.c_uint32),
                ("rev_long", C.c_uint32), ("sb_shift", C.c_uint32), ("tile_ticket", C.c_uint32 * 8),
                ("digit_of_slot", C.c_int32 * 8), ("src_of_slot", C.c_int32 * 8), ("dst_of_slot", C.c_int32 * 8),
                ("prof", C.c_uint64 * 16)]


off = RadixState.prof.offset
acc = temp[off:off + 128].cpu().numpy().view(np.uint64)
tiles = int(acc[3])
print(f"tiles={tiles}  cycles/tile: phase1={acc[0] / tiles:.0f}  totals+lookback={acc[1] / tiles:.0f}"
      f"  bases+phase2={acc[2] / tiles:.0f}")
# k_onesweep_t (radix_onesweep_tma.cuh): count, per-digit section, rank, write-out; inside the section: copy wait, totals + look-back
print("k_onesweep_t cycles/tile: " + "  ".join(
    f"{name}={acc[i] / tiles:.0f}" for name, i in (("count", 0), ("digit_section", 1), ("rank", 2), ("write_out", 4),
                                                   ("copy_wait", 5), ("totals_lookback", 6), ("totals", 7))))

if acc[11]:
    print(f"look-back of digit 0 per walk: rounds={acc[8] / acc[11]:.2f}  blocked rounds={acc[9] / acc[11]:.2f}"
          f"  tiles consumed before the last round={acc[10] / acc[11]:.1f}")
