"""ctypes access to the parity checker.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module.  It exposes
  * ``Oracle``    -- oracle/liboracle.so, our C restatement (isort_oracle.c), and
  * ``Reference`` -- oracle/_ref/libintsort_ref.so, the unmodified reference
                     library compiled from /root/reference (present only where it
                     was built; it travels to the GPU box prebuilt).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libintsort_ref.so")
RECORD_DTYPE = np.dtype([("key", "<u8"), ("tag", "<u8")])

_u64, _u32, _i32, _vp, _dbl = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_void_p, ctypes.c_double


class OracleError(ValueError):
    pass


def _p(a: np.ndarray):
    return a.ctypes.data if a.size else None


def _recs(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a))
    if a.dtype != RECORD_DTYPE:
        raise TypeError("expected records")
    return a


class Oracle:
    """Our C restatement of the reference algorithm (oracle/isort_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = self.lib = ctypes.CDLL(path)
        sig = {
            "orc_last_error": (ctypes.c_char_p, []),
            "orc_mix64": (_u64, [_u64]),
            "orc_splitmix_next": (_u64, [ctypes.POINTER(_u64)]),
            "orc_splitmix_below": (_i32, [ctypes.POINTER(_u64), _u64, ctypes.POINTER(_u64)]),
            "orc_default_range_bound": (_u64, [_i32]),
            "orc_generate": (_i32, [_i32, _u64, _i32, _u64, _u64, _i32, _u64, _dbl, _vp]),
            "orc_gen_uniform_u32": (None, [_u64, _u64, _u32, _vp]),
            "orc_gen_mixture_u32": (None, [_u64, _u64, _vp]),
            "orc_gen_mixture_u32_range": (None, [_u64, _u64, _u64, _vp]),
            "orc_insertion_sort": (None, [_vp, _vp, _u64]),
            "orc_extract_digit": (_i32, [_u64, _u32, _u64, ctypes.POINTER(_u64)]),
            "orc_build_radix_plan": (_i32, [_vp, _u64, _u64, ctypes.POINTER(_u32)]),
            "orc_counting_sort_by_digit": (_i32, [_vp, _vp, _u64, _u64, _u32, _u32]),
            "orc_radix_sort_lsd": (_i32, [_vp, _vp, _u64, _u64]),
            "orc_bucket_index": (_i32, [_u64, _u64, _u64, ctypes.POINTER(_u64)]),
            "orc_bucket_sort": (_i32, [_vp, _vp, _u64, _u64, ctypes.POINTER(_u64)]),
            "orc_oracle_sort": (_i32, [_vp, _vp, _u64]),
            "orc_is_sorted": (_i32, [_vp, _u64]),
            "orc_radix_sort_u32": (_i32, [_vp, _vp, _vp, _vp, _u64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args

    def _chk(self, rc: int) -> None:
        if rc:
            raise OracleError(self.lib.orc_last_error().decode())

    # rng / generator (rng.hpp, generator.cpp)
    def splitmix_stream(self, seed: int, count: int) -> list[int]:
        st = _u64(seed)
        return [int(self.lib.orc_splitmix_next(ctypes.byref(st))) for _ in range(count)]

    def default_range_bound(self, case_id: int) -> int:
        return int(self.lib.orc_default_range_bound(case_id))

    def write_sequence_file(self, path: str, header: tuple, records: np.ndarray) -> None:
        """The reference's write_sequence_file (sequence_io.cpp:63-70); header = (case_id, n, M, seed)."""
        h = (ctypes.c_uint64 * 4)(*header)
        rec = np.ascontiguousarray(records, dtype=RECORD_DTYPE)
        self._chk(self.lib.ref_write_sequence_file(os.fsencode(path), h, rec.ctypes.data, rec.size))

    def read_sequence_file(self, path: str, capacity: int = 1 << 20):
        """The reference's read_sequence_file: ((case_id, n, M, seed), records) or
        OracleError with the reference's SequenceIoError message."""
        h = (ctypes.c_uint64 * 4)()
        out = np.empty(capacity, dtype=RECORD_DTYPE)
        self._chk(self.lib.ref_read_sequence_file(os.fsencode(path), h, out.ctypes.data, capacity))
        return tuple(int(x) for x in h), out[: h[1]].copy()

    def generate(self, case_id: int, n: int, range_bound: int | None = None, seed: int = 0,
                 repeated_value: int | None = None, sorted_fraction: float = 0.95) -> np.ndarray:
        out = np.empty(n, dtype=RECORD_DTYPE)
        self._chk(self.lib.orc_generate(case_id, n, range_bound is not None, range_bound or 0, seed,
                                        repeated_value is not None, repeated_value or 0, sorted_fraction,
                                        _p(out)))
        return out

    def uniform_u32(self, n: int, seed: int = 42, bits: int = 32) -> np.ndarray:
        out = np.empty(n, dtype=np.uint32)
        self.lib.orc_gen_uniform_u32(n, seed, bits, _p(out))
        return out

    def mixture_u32(self, n: int, seed: int = 42, threads: int | None = None) -> np.ndarray:
        """Config-5 keys; large n is split over host threads (ctypes drops the GIL),
        each writing its own index range -- the same values as one sequential call."""
        out = np.empty(n, dtype=np.uint32)
        threads = threads or (min(os.cpu_count() or 1, 32) if n >= (1 << 22) else 1)
        if threads <= 1:
            self.lib.orc_gen_mixture_u32(n, seed, _p(out))
            return out
        import threading

        step = (n + threads - 1) // threads
        def part(s):
            c = min(step, n - s)
            if c > 0:
                self.lib.orc_gen_mixture_u32_range(s, c, seed, out.ctypes.data + 4 * s)
        ths = [threading.Thread(target=part, args=(s,)) for s in range(0, n, step)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return out

    # sorting core (sort.cpp)
    def insertion_sort(self, seq) -> np.ndarray:
        a = _recs(seq)
        out = np.empty_like(a)
        self.lib.orc_insertion_sort(_p(a), _p(out), a.size)
        return out

    def extract_digit(self, key: int, digit_index: int, base: int) -> int:
        r = _u64(0)
        self._chk(self.lib.orc_extract_digit(key, digit_index, base, ctypes.byref(r)))
        return int(r.value)

    def build_radix_plan(self, seq, base: int) -> int:
        a = _recs(seq)
        d = _u32(0)
        self._chk(self.lib.orc_build_radix_plan(_p(a), a.size, base, ctypes.byref(d)))
        return int(d.value)

    def counting_sort_by_digit(self, seq, base: int, digits: int, digit_index: int) -> np.ndarray:
        a = _recs(seq)
        out = np.empty_like(a)
        self._chk(self.lib.orc_counting_sort_by_digit(_p(a), _p(out), a.size, base, digits, digit_index))
        return out

    def radix_sort_lsd(self, seq, base: int = 10) -> np.ndarray:
        a = _recs(seq)
        out = np.empty_like(a)
        self._chk(self.lib.orc_radix_sort_lsd(_p(a), _p(out), a.size, base))
        return out

    def bucket_index(self, key: int, count: int, range_bound: int) -> int:
        r = _u64(0)
        self._chk(self.lib.orc_bucket_index(key, count, range_bound, ctypes.byref(r)))
        return int(r.value)

    def bucket_sort(self, seq, range_bound: int) -> np.ndarray:
        a = _recs(seq)
        out = np.empty_like(a)
        bad = _u64(0)
        self._chk(self.lib.orc_bucket_sort(_p(a), _p(out), a.size, range_bound, ctypes.byref(bad)))
        return out

    def oracle_sort(self, seq) -> np.ndarray:
        a = _recs(seq)
        out = np.empty_like(a)
        self._chk(self.lib.orc_oracle_sort(_p(a), _p(out), a.size))
        return out

    def sort_u32(self, keys: np.ndarray, with_index: bool = False):
        """Stable LSD sort of u32 keys (+ original positions): the keys-only
        restatement of radix_sort_lsd at base 256, for BASELINE-sized parity."""
        k = np.ascontiguousarray(keys, dtype=np.uint32)
        ko = np.empty_like(k)
        vo = np.empty_like(k) if with_index else None
        self._chk(self.lib.orc_radix_sort_u32(_p(k), _p(ko), None, _p(vo) if vo is not None else None, k.size))
        return (ko, vo) if with_index else ko


class Reference:
    """The unmodified reference library (oracle/_ref/libintsort_ref.so)."""

    ALG = {"bucket": 0, "radix": 1, "insertion": 2}  # AlgorithmId order, bench.hpp:15

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: it is built by `make -C oracle ref` where /root/reference exists")
        L = self.lib = ctypes.CDLL(path)
        sig = {
            "ref_last_error": (ctypes.c_char_p, []),
            "ref_radix_sort_lsd": (_i32, [_vp, _vp, _u64, _u64]),
            "ref_bucket_sort": (_i32, [_vp, _vp, _u64, _u64]),
            "ref_insertion_sort": (_i32, [_vp, _vp, _u64]),
            "ref_counting_sort_by_digit": (_i32, [_vp, _vp, _u64, _u64, _u32, _u32]),
            "ref_build_radix_plan": (_i32, [_vp, _u64, _u64, ctypes.POINTER(_u32)]),
            "ref_extract_digit": (_i32, [_u64, _u32, _u64, ctypes.POINTER(_u64)]),
            "ref_bucket_index": (_i32, [_u64, _u64, _u64, ctypes.POINTER(_u64)]),
            "ref_oracle_sort": (_i32, [_vp, _vp, _u64]),
            "ref_generate": (_i32, [_i32, _u64, _i32, _u64, _u64, _i32, _u64, _dbl, _vp]),
            "ref_splitmix_next": (_u64, [_u64, _u64]),
            "ref_write_sequence_file": (_i32, [ctypes.c_char_p, ctypes.POINTER(_u64), _vp, _u64]),
            "ref_read_sequence_file": (_i32, [ctypes.c_char_p, ctypes.POINTER(_u64), _vp, _u64]),
            "ref_time_one": (_dbl, [_i32, _vp, _u64, _u64, _u64]),
            "ref_time_sort": (_i32, [_i32, _vp, _u64, _u64, _u64, _i32, ctypes.POINTER(_dbl),
                                     ctypes.POINTER(_dbl)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args

    def _chk(self, rc: int) -> None:
        if rc:
            raise OracleError(self.lib.ref_last_error().decode())

    def write_sequence_file(self, path: str, header: tuple, records: np.ndarray) -> None:
        """The reference's write_sequence_file (sequence_io.cpp:63-70); header = (case_id, n, M, seed)."""
        h = (ctypes.c_uint64 * 4)(*header)
        rec = np.ascontiguousarray(records, dtype=RECORD_DTYPE)
        self._chk(self.lib.ref_write_sequence_file(os.fsencode(path), h, rec.ctypes.data, rec.size))

    def read_sequence_file(self, path: str, capacity: int = 1 << 20):
        """The reference's read_sequence_file: ((case_id, n, M, seed), records) or
        OracleError with the reference's SequenceIoError message."""
        h = (ctypes.c_uint64 * 4)()
        out = np.empty(capacity, dtype=RECORD_DTYPE)
        self._chk(self.lib.ref_read_sequence_file(os.fsencode(path), h, out.ctypes.data, capacity))
        return tuple(int(x) for x in h), out[: h[1]].copy()

    def generate(self, case_id: int, n: int, range_bound: int | None = None, seed: int = 0,
                 repeated_value: int | None = None, sorted_fraction: float = 0.95) -> np.ndarray:
        out = np.empty(n, dtype=RECORD_DTYPE)
        self._chk(self.lib.ref_generate(case_id, n, range_bound is not None, range_bound or 0, seed,
                                        repeated_value is not None, repeated_value or 0, sorted_fraction,
                                        _p(out)))
        return out

    def radix_sort_lsd(self, seq, base: int = 10) -> np.ndarray:
        a = _recs(seq)
        out = np.empty_like(a)
        self._chk(self.lib.ref_radix_sort_lsd(_p(a), _p(out), a.size, base))
        return out

    def bucket_sort(self, seq, range_bound: int) -> np.ndarray:
        a = _recs(seq)
        out = np.empty_like(a)
        self._chk(self.lib.ref_bucket_sort(_p(a), _p(out), a.size, range_bound))
        return out

    def counting_sort_by_digit(self, seq, base: int, digits: int, digit_index: int) -> np.ndarray:
        a = _recs(seq)
        out = np.empty_like(a)
        self._chk(self.lib.ref_counting_sort_by_digit(_p(a), _p(out), a.size, base, digits, digit_index))
        return out

    def build_radix_plan(self, seq, base: int) -> int:
        a = _recs(seq)
        d = _u32(0)
        self._chk(self.lib.ref_build_radix_plan(_p(a), a.size, base, ctypes.byref(d)))
        return int(d.value)

    def bucket_index(self, key: int, count: int, range_bound: int) -> int:
        r = _u64(0)
        self._chk(self.lib.ref_bucket_index(key, count, range_bound, ctypes.byref(r)))
        return int(r.value)

    def oracle_sort(self, seq) -> np.ndarray:
        a = _recs(seq)
        out = np.empty_like(a)
        self._chk(self.lib.ref_oracle_sort(_p(a), _p(out), a.size))
        return out

    def time_one(self, algorithm: str, seq, range_bound: int, base: int) -> float:
        a = _recs(seq)
        t = self.lib.ref_time_one(self.ALG[algorithm], _p(a), a.size, range_bound, base)
        if t < 0:
            raise OracleError(self.lib.ref_last_error().decode())
        return t
