"""CPU checks of the C-ABI boundary: the library loads, exports every symbol
include/isort.h declares, carries sm_100a code, validates arguments the way the
reference does, and fails loudly (no CPU fallback) when no GPU is present."""
from __future__ import annotations

import ctypes
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

from paper_1206_3511_b200 import _lib
import paper_1206_3511_b200 as isort

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "isort.h")


def declared_functions() -> list[str]:
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(isort_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("isort_radix_sort_u32", "isort_bucket_sort_u32", "isort_radix_sort_records",
                 "isort_bucket_sort_records", "isort_counting_sort_by_digit_records",
                 "isort_build_radix_plan_records", "isort_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} missing from the ctypes signature table"


@pytest.mark.skipif(shutil.which("cuobjdump") is None and not os.path.exists("/usr/local/cuda/bin/cuobjdump"),
                    reason="cuobjdump not available")
def test_library_is_sm100a_native():
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([tool, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out


def test_abi_version_and_limits():
    lib = _lib.load()
    assert lib.isort_abi_version() == 1
    assert lib.isort_max_keys() == (1 << 32) - 1


def test_reference_argument_errors_without_device():
    # base < 2 is rejected before any device work (sort.cpp:58-60), even for empty input
    with pytest.raises(isort.InvalidArgument, match="base must be >= 2"):
        isort.radix_sort_lsd(isort.seq_of([]), 1)
    with pytest.raises(isort.InvalidArgument, match="base must be >= 2"):
        isort.build_radix_plan(isort.seq_of([1]), 1)
    with pytest.raises(isort.InvalidArgument, match="out of range for a 3-digit plan"):
        isort.counting_sort_by_digit(isort.seq_of([170, 45, 75]), isort.RadixPlan(10, 3), 3)
    with pytest.raises(isort.InvalidArgument, match="base must be >= 2"):
        isort.extract_digit(1, 0, 1)
    # empty input: bucket_sort returns empty without a range check (sort.cpp:139-141)
    assert isort.bucket_sort(isort.seq_of([]), 0).size == 0
    assert isort.radix_sort_lsd(isort.seq_of([]), 10).size == 0


def test_extract_digit_scalar():
    assert [isort.extract_digit(170, i, 10) for i in range(4)] == [0, 7, 1, 0]


def test_no_cpu_fallback_when_no_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(isort.CudaError, match="no CPU fallback"):
        isort.radix_sort_lsd(isort.seq_of([3, 1, 2]), 10)
    with pytest.raises(isort.CudaError):
        isort.bucket_sort(isort.seq_of([3, 1, 2]), 10)


def test_device_entry_points_validate_arguments():
    lib = _lib.load()
    # bad vals_mode and undersized temp are argument errors (no device touched)
    rc = lib.isort_radix_sort_u32(None, None, None, None, 10, 7, None, 0, None)
    assert rc == _lib.ISORT_EINVAL
    rc = lib.isort_radix_sort_u32(ctypes.c_void_p(16), ctypes.c_void_p(16), None, None, 10, 0, None, 0, None)
    assert rc == _lib.ISORT_EINVAL and b"temp buffer too small" in lib.isort_last_error()
    rc = lib.isort_radix_sort_u32(ctypes.c_void_p(16), ctypes.c_void_p(16), None, None, 1 << 32, 0, None, 0, None)
    assert rc == _lib.ISORT_ERANGE
    assert lib.isort_radix_temp_bytes(10**8, 4, 0) > 4 * 10**8
    assert lib.isort_bucket_temp_bytes(10**8, 4, 2) > lib.isort_radix_temp_bytes(10**8, 4, 2)
    assert lib.isort_bucket_index_u64(None, None, 1, 0, 5, None) == _lib.ISORT_EINVAL


def test_record_layout_matches_reference():
    assert isort.RECORD_DTYPE.itemsize == 16
    s = isort.seq_of([5, 4])
    assert s["tag"].tolist() == [0, 1]
    assert np.asarray(s).view(np.uint64).tolist() == [5, 0, 4, 1]
