"""Build an A/B variant of libisort.so: the named translation units recompiled
with extra nvcc flags, every other unit taken from the default build.

    python tools/build_variant.py NAME "-DISORT_UF_REP=16" inst_radix_u32 [more units]
    -> tools/ab/NAME/libisort.so   (time it with tools/ab_block.py)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1206_3511_b200 import _build  # noqa: E402

name, flags, units = sys.argv[1], sys.argv[2].split(), sys.argv[3:]
out = os.path.join(ROOT, "tools", "ab", name)
os.makedirs(out, exist_ok=True)
_build.build_engine()
objs = []
for o in sorted(os.listdir(_build.OBJ_DIR)):
    if not o.endswith(".o"):
        continue
    unit = o[:-2]
    if unit in units:
        dst = os.path.join(out, o)
        subprocess.run([_build._nvcc(), *_build.NVCC_FLAGS, *flags, "-c", "-o", dst,
                        os.path.join(_build.CSRC, unit + ".cu")], check=True)
        objs.append(dst)
    else:
        objs.append(os.path.join(_build.OBJ_DIR, o))
subprocess.run([_build._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xlinker", "--no-undefined",
                "-o", os.path.join(out, "libisort.so"), *objs], check=True)
print(os.path.join(out, "libisort.so"))
