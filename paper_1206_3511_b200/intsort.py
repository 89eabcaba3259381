"""Python mirror of the reference's sorting API (proj/core/include/intsort/sort.hpp).

Same names, argument meaning and error behaviour as the C++ library, so the
parity tests read like proj/tests/test_sort.cpp.  A ``RecordSeq`` is a numpy
structured array with the reference's 16-byte layout ``{u64 key, u64 tag}``
(record.hpp:20-25).  Every sort runs on the B200 through the C ABI
(include/isort.h); there is no CPU fallback -- without a GPU the calls raise
:class:`CudaError`.  ``std::invalid_argument`` maps to :class:`InvalidArgument`
(a ``ValueError``).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import CudaError, InvalidArgument, IsortError  # noqa: F401  (re-exported)

RECORD_DTYPE = np.dtype([("key", "<u8"), ("tag", "<u8")])
K_MAX_RANGE_BOUND = 1 << 40  # record.hpp:15


def seq_of(keys) -> np.ndarray:
    """Records from bare keys, tag = original position (proj/tests/helpers.hpp:11-19)."""
    k = np.asarray(list(keys) if not isinstance(keys, np.ndarray) else keys, dtype=np.uint64).reshape(-1)
    out = np.empty(k.shape[0], dtype=RECORD_DTYPE)
    out["key"] = k
    out["tag"] = np.arange(k.shape[0], dtype=np.uint64)
    return out


def keys_of(seq: np.ndarray) -> list[int]:
    return [int(x) for x in seq["key"]]


def tags_of(seq: np.ndarray) -> list[int]:
    return [int(x) for x in seq["tag"]]


def as_record_seq(seq) -> np.ndarray:
    a = np.asarray(seq)
    if a.dtype != RECORD_DTYPE:
        raise TypeError(f"expected a RecordSeq ({RECORD_DTYPE}), got {a.dtype}")
    return np.ascontiguousarray(a)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


@dataclass
class RadixPlan:
    """sort.hpp:13-16."""

    base: int = 10
    digits: int = 1


def _device() -> int:
    return 0


def radix_sort_lsd(seq, base: int = 10) -> np.ndarray:
    """Stable LSD radix sort (sort.hpp:37-40).  Output identical for every base >= 2;
    throws on base < 2 (sort.cpp:58-60) even for empty input."""
    a = as_record_seq(seq)
    out = np.empty_like(a)
    lib = _lib.load()
    _lib.check(lib.isort_radix_sort_records(_ptr(a), _ptr(out), a.shape[0], int(base), _device()))
    return out


def bucket_sort(seq, range_bound: int) -> np.ndarray:
    """n-bucket distribution sort (sort.hpp:50-53).  Empty input returns empty
    without a range check (sort.cpp:139-141); a key > range_bound raises."""
    a = as_record_seq(seq)
    out = np.empty_like(a)
    lib = _lib.load()
    _lib.check(lib.isort_bucket_sort_records(_ptr(a), _ptr(out), a.shape[0], int(range_bound), _device()))
    return out


def insertion_sort(seq) -> np.ndarray:
    """Stable sort by key (sort.hpp:18-21).  The quadratic loop is the reference's
    cost model, not its contract: the unique stable output comes from the device."""
    return radix_sort_lsd(seq, 256)


def build_radix_plan(seq, base: int) -> RadixPlan:
    """Minimal digits with base^digits > max key (sort.hpp:28, sort.cpp:57-75)."""
    a = as_record_seq(seq)
    d = ctypes.c_uint32(0)
    lib = _lib.load()
    _lib.check(lib.isort_build_radix_plan_records(_ptr(a), a.shape[0], int(base), ctypes.byref(d), _device()))
    return RadixPlan(int(base), int(d.value))


def counting_sort_by_digit(seq, plan: RadixPlan, digit_index: int) -> np.ndarray:
    """One stable counting pass on digit `digit_index` (sort.hpp:30-35)."""
    a = as_record_seq(seq)
    out = np.empty_like(a)
    lib = _lib.load()
    _lib.check(lib.isort_counting_sort_by_digit_records(_ptr(a), _ptr(out), a.shape[0], int(plan.base),
                                                         int(plan.digits), int(digit_index), _device()))
    return out


def extract_digit(key: int, digit_index: int, base: int) -> int:
    """floor(key / base^digit_index) mod base by repeated division (sort.cpp:44-55).
    A scalar helper, not a data-parallel path: plain integer arithmetic."""
    if base < 2:
        raise InvalidArgument(_lib.ISORT_EINVAL, "extract_digit: base must be >= 2")
    v = int(key)
    i = 0
    while i < digit_index and v != 0:
        v //= base
        i += 1
    return v % base


def bucket_index_batch(keys, bucket_count: int, range_bound: int) -> np.ndarray:
    """Device batch of bucket_index (sort.cpp:121-134); raises like the reference
    for bucket_count == 0 or the first key > range_bound."""
    import torch  # device memory plumbing

    k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64).reshape(-1))
    if bucket_count == 0:
        raise InvalidArgument(_lib.ISORT_EINVAL, "bucket_index: bucket_count must be >= 1")
    if k.size == 0:
        return np.zeros(0, dtype=np.uint64)
    if not torch.cuda.is_available():
        raise CudaError(_lib.ISORT_ECUDA, "no CUDA device available; the engine has no CPU fallback")
    dk = torch.from_numpy(k.view(np.int64)).cuda()
    dout = torch.empty_like(dk)
    lib = _lib.load()
    stream = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.isort_bucket_index_u64(dk.data_ptr(), dout.data_ptr(), k.size, int(bucket_count),
                                          int(range_bound), stream))
    out = dout.cpu().numpy().view(np.uint64)
    bad = np.nonzero(out == np.uint64(0xFFFFFFFFFFFFFFFF))[0]
    if bad.size:
        key = int(k[bad[0]])
        raise InvalidArgument(_lib.ISORT_EINVAL,
                              f"bucket_index: key {key} exceeds range bound {int(range_bound)} "
                              "(sequence/spec mismatch)")
    return out


def bucket_index(key: int, bucket_count: int, range_bound: int) -> int:
    """floor(bucket_count * key / (range_bound + 1)) (sort.hpp:42-48), on the device."""
    return int(bucket_index_batch([key], bucket_count, range_bound)[0])
