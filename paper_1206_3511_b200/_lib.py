"""ctypes binding of libisort.so (the C ABI declared in include/isort.h).

The shared library is built in-tree by :mod:`paper_1206_3511_b200._build`
(``nvcc -gencode arch=compute_100a,code=sm_100a``).  There is no CPU fallback:
if the library is missing, loading fails loudly; if no CUDA device is present,
every sorting call returns ``ISORT_ECUDA`` and raises :class:`CudaError`.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libisort.so")

ISORT_OK = 0
ISORT_ENOMEM = 12
ISORT_EINVAL = 22
ISORT_ERANGE = 34
ISORT_EIO = 5
ISORT_ECUDA = 1001
ISORT_ENCCL = 1002

VALS_NONE = 0
VALS_LOAD = 1
VALS_IOTA = 2

# name -> (restype, argtypes); mirrors include/isort.h one to one.
_u64, _u32, _i32, _sz = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_size_t
_vp = ctypes.c_void_p


class SequenceHeaderC(ctypes.Structure):
    """isort_sequence_header (include/isort.h): the ISRT header fields."""
    _fields_ = [("case_id", _u64), ("n", _u64), ("range_bound", _u64), ("seed", _u64)]


SIGNATURES = {
    "isort_last_error": (ctypes.c_char_p, []),
    "isort_abi_version": (_i32, []),
    "isort_max_keys": (_u64, []),
    "isort_last_bad_index": (_u64, []),
    "isort_launch_count": (_u64, []),
    "isort_rank_mode": (_i32, []),
    "isort_init": (_i32, [_i32]),
    "isort_pool_trim": (_i32, [_i32]),
    "isort_profile_begin": (_i32, []),
    "isort_profile_end": (_i32, [ctypes.POINTER(ctypes.c_float), ctypes.c_char_p, _i32, _i32,
                                 ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
    "isort_radix_temp_bytes": (_sz, [_u64, _i32, _i32]),
    "isort_radix_sort_u32": (_i32, [_vp, _vp, _vp, _vp, _u64, _i32, _vp, _sz, _vp]),
    "isort_radix_sort_u64": (_i32, [_vp, _vp, _vp, _vp, _u64, _i32, _vp, _sz, _vp]),
    "isort_bucket_temp_bytes": (_sz, [_u64, _i32, _i32]),
    "isort_bucket_sort_u32": (_i32, [_vp, _vp, _vp, _vp, _u64, _u64, _i32, _vp, _sz, _vp]),
    "isort_bucket_sort_u64": (_i32, [_vp, _vp, _vp, _vp, _u64, _u64, _i32, _vp, _sz, _vp]),
    "isort_bucket_sort_span_u32": (_i32, [_vp, _vp, _vp, _vp, _u64, _u64, _u64, _i32, _vp, _sz, _vp]),
    "isort_counting_pass_temp_bytes": (_sz, [_u64]),
    "isort_counting_pass_u32": (_i32, [_vp, _vp, _vp, _vp, _u64, _u64, _u32, _u32, _i32, _vp, _sz, _vp]),
    "isort_partition_temp_bytes": (_sz, [_u64, _i32, _i32]),
    "isort_partition_u32": (_i32, [_vp, _vp, _vp, _vp, _u64, _vp, _i32, _i32, _vp, _vp, _sz, _vp]),
    "isort_radix_sort_records": (_i32, [_vp, _vp, _u64, _u64, _i32]),
    "isort_bucket_sort_records": (_i32, [_vp, _vp, _u64, _u64, _i32]),
    "isort_counting_sort_by_digit_records": (_i32, [_vp, _vp, _u64, _u64, _u32, _u32, _i32]),
    "isort_build_radix_plan_records": (_i32, [_vp, _u64, _u64, ctypes.POINTER(_u32), _i32]),
    "isort_radix_sort_host_u32": (_i32, [_vp, _vp, _u64, _i32]),
    "isort_bucket_sort_host_u32": (_i32, [_vp, _vp, _u64, _u64, _i32]),
    "isort_is_sorted_u32": (_i32, [_vp, _u64, ctypes.POINTER(_i32), _vp]),
    "isort_bucket_index_u64": (_i32, [_vp, _vp, _u64, _u64, _u64, _vp]),
    "isort_bucket_sort_u32_async": (_i32, [_vp, _vp, _vp, _vp, _u64, _u64, _i32, _vp, _sz, _vp, _vp]),
    "isort_bucket_finish_u32": (_i32, [_vp, _vp, _vp, _u64, _u64, _i32, _vp, _sz, _vp, _vp]),
    "isort_partition_counts_u32": (_i32, [_vp, _u64, _vp, _i32, _vp, _vp, _sz, _vp]),
    "isort_partition_scatter_u32": (_i32, [_vp, _vp, _u64, _vp, _i32, _i32, _vp, _vp, _vp, _sz, _vp]),
    "isort_partition_scatter_table_u32": (_i32, [_vp, _vp, _u64, _vp, _i32, _i32, _vp, _vp, _sz, _vp]),
    "isort_ipc_alloc": (_i32, [_sz, _i32, ctypes.POINTER(_vp), _vp]),
    "isort_ipc_open": (_i32, [_vp, _i32, ctypes.POINTER(_vp)]),
    "isort_ipc_close": (_i32, [_vp]),
    "isort_ipc_free": (_i32, [_vp]),
    "isort_sequence_read_header": (_i32, [ctypes.c_char_p, ctypes.POINTER(SequenceHeaderC)]),
    "isort_sequence_load": (_i32, [ctypes.c_char_p, _vp, _u64, _i32, ctypes.POINTER(SequenceHeaderC), _i32]),
}


class IsortError(RuntimeError):
    """Base class for engine errors (non-zero ISORT_* status)."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


class InvalidArgument(IsortError, ValueError):
    """ISORT_EINVAL: the reference throws std::invalid_argument here."""


class SequenceIoError(IsortError):
    """ISORT_EIO: the reference throws intsort::SequenceIoError here (sequence_io.hpp:31-33)."""


class CudaError(IsortError):
    """ISORT_ECUDA: no device, or a CUDA call failed.  Never silently retried on CPU."""


_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load libisort.so once; raise if it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(the engine has no CPU fallback)"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(code: int) -> None:
    """Raise the Python mirror of an ISORT_* status."""
    if code == ISORT_OK:
        return
    msg = load().isort_last_error().decode("utf-8", "replace")
    if code == ISORT_EINVAL:
        raise InvalidArgument(code, msg)
    if code == ISORT_ECUDA:
        raise CudaError(code, msg)
    if code == ISORT_EIO:
        raise SequenceIoError(code, msg)
    raise IsortError(code, msg)


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
