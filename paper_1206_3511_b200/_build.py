"""In-tree build of the engine (and of the parity checker under oracle/).

* ``libisort.so``: every CUDA translation unit in csrc/ compiled for sm_100a only
  (``-gencode arch=compute_100a,code=sm_100a``), ``-lineinfo`` so ncu's source
  page maps to our code.  Built next to this file so it travels to the GPU box
  with the repo snapshot.
* ``oracle/liboracle.so`` (the C restatement) and, where /root/reference
  exists, ``oracle/_ref/*`` (the reference itself) -- test infrastructure only.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
import time

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libisort.so")
REFERENCE = "/root/reference/proj"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    # (no -split-compile: measured 62.8 vs 81.3 Gkeys/s for the radix sort -- it changes the kernels' code;
    #  the kernels are split across translation units instead, see csrc/isort_launch.cuh)
]
OBJ_DIR = os.path.join(PKG, "build")


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a engine (no CPU fallback exists)")


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_engine(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    """Compile every translation unit of csrc/ to an object (in parallel: ptxas
    is single-threaded per unit), then link libisort.so.  --no-undefined makes a
    missing explicit instantiation a build error rather than a load error."""
    from concurrent.futures import ThreadPoolExecutor

    units = sorted(glob.glob(os.path.join(CSRC, "*.cu")))  # translation units of libisort.so
    headers = sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
                     + [os.path.join(ROOT, "include", "isort.h")])
    os.makedirs(OBJ_DIR, exist_ok=True)
    objs = [os.path.join(OBJ_DIR, os.path.basename(u)[:-3] + ".o") for u in units]
    todo = [(u, o) for u, o in zip(units, objs) if force or _stale(o, [u] + headers)]

    def compile_one(uo):
        u, o = uo
        cmd = [_nvcc(), *NVCC_FLAGS, "-c", "-o", o + ".tmp", u]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        t0 = time.time()
        subprocess.run(cmd, check=True, cwd=CSRC)
        os.replace(o + ".tmp", o)
        os.utime(o, (t0, t0))  # a source edited while this unit compiled still counts as newer

    if todo:
        with ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
            list(ex.map(compile_one, todo))
    if force or todo or _stale(LIB, objs):
        cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xlinker", "--no-undefined",
               "-o", LIB + ".tmp", *objs]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True, cwd=CSRC)
        os.replace(LIB + ".tmp", LIB)
    return LIB


def build_oracle(verbose: bool = False) -> None:
    """Build the checker: our restatement always, the reference where it exists."""
    oracle = os.path.join(ROOT, "oracle")
    targets = ["oracle"]
    if os.path.isdir(REFERENCE):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", oracle, *targets], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)


def build_dropin(verbose: bool = False) -> None:
    """The C++ drop-in (dropin/sort_b200.cpp) linked with the reference's other
    sources and its own test suites -- only where /root/reference exists; the
    binaries travel to the GPU box prebuilt under oracle/_ref/."""
    if not os.path.isdir(REFERENCE):
        return
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "dropin"], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_engine(force=force, verbose=verbose)
    build_oracle(verbose=verbose)
    build_dropin(verbose=verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose=True)
