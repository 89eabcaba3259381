"""Device-resident sorts over torch tensors (torch is plumbing: memory + streams).

Keys are u32 or u64 bit patterns held in ``torch.int32`` / ``torch.int64``
(or ``torch.uint32`` / ``torch.uint64``) CUDA tensors; payloads are 32-bit.
Each call goes straight to the C ABI (include/isort.h) on the current torch
stream.  :class:`Sorter` keeps its output and temp buffers so repeated calls
(benchmarks) allocate nothing.
"""
from __future__ import annotations

import torch

from . import _lib

_U32 = {torch.int32, getattr(torch, "uint32", torch.int32)}
_U64 = {torch.int64, getattr(torch, "uint64", torch.int64)}

RADIX = "radix"
BUCKET = "bucket"


def _key_bytes(t: torch.Tensor) -> int:
    if t.dtype in _U32:
        return 4
    if t.dtype in _U64:
        return 8
    raise TypeError(f"keys must be 32- or 64-bit integer tensors, got {t.dtype}")


def _check_cuda(t: torch.Tensor, what: str) -> None:
    if not t.is_cuda:
        raise _lib.CudaError(_lib.ISORT_ECUDA, f"{what} must be a CUDA tensor (the engine has no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")


class Sorter:
    """Reusable device sort of n keys (+ optional u32 payload).

    ``vals``: None (keys only), "iota" (payload = original position, generated on
    the device) or "load" (a payload tensor is passed to :meth:`__call__`).

    ``graph=True``: the first call with a given input runs eagerly, the second
    captures the whole pipeline (state reset, histogram, plan, passes, copy; for
    the bucket sort also the segment sort and its status) into a CUDA graph, and
    later calls with the same input and payload tensors replay it -- one launch
    instead of ~10, which is what small, latency-bound sorts pay for.  The bucket
    sort's status comes back through host-pinned memory
    (isort_bucket_sort_u32_async) and is checked after the replay
    (isort_bucket_finish_u32: range error, oversized fallback).

    ``range_lo`` (bucket, u32 keys): the buckets cover [range_lo, range_bound]
    instead of [0, range_bound] (isort_bucket_sort_span_u32) -- the multi-GPU
    local sort, where a rank holds one key range.  Eager only.
    """

    def __init__(self, n: int, key_bytes: int = 4, algorithm: str = RADIX, vals: str | None = None,
                 range_bound: int | None = None, device: torch.device | str = "cuda", graph: bool = False,
                 range_lo: int = 0):
        if algorithm not in (RADIX, BUCKET):
            raise ValueError(f"unknown algorithm {algorithm!r}")
        if algorithm == BUCKET and range_bound is None:
            range_bound = (1 << (8 * key_bytes)) - 1
        if range_lo and (algorithm != BUCKET or key_bytes != 4):
            raise ValueError("range_lo applies to the u32 bucket sort only")
        self.n, self.key_bytes, self.algorithm, self.range_bound = n, key_bytes, algorithm, range_bound
        self.range_lo = int(range_lo)
        self.vmode = {None: _lib.VALS_NONE, "load": _lib.VALS_LOAD, "iota": _lib.VALS_IOTA}[vals]
        lib = _lib.load()
        tb = (lib.isort_radix_temp_bytes if algorithm == RADIX else lib.isort_bucket_temp_bytes)(
            n, key_bytes, self.vmode)
        dt = torch.int32 if key_bytes == 4 else torch.int64
        self.device = torch.device(device)
        self.keys_out = torch.empty(max(n, 1), dtype=dt, device=self.device)[:n]
        self.vals_out = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)[:n] if vals else None
        self.temp = torch.empty(max(tb, 1), dtype=torch.uint8, device=self.device)
        self.temp_bytes = tb
        # graphs need the lane-ordered rank (the fallback synchronises inside the bucket sort)
        self.graph = (graph and (algorithm == RADIX or key_bytes == 4) and not self.range_lo
                      and lib.isort_rank_mode() != 0)
        self._status = (torch.zeros(32, dtype=torch.uint8, pin_memory=True)
                        if self.graph and algorithm == BUCKET else None)
        self._graph = None
        self._graph_key = None
        self.launches_per_call = None  # kernels in the captured pipeline

    def __call__(self, keys: torch.Tensor, vals_in: torch.Tensor | None = None, stream=None, eager: bool = False):
        _check_cuda(keys, "keys")
        if keys.numel() != self.n or _key_bytes(keys) != self.key_bytes:
            raise ValueError("keys do not match the Sorter's shape/width")
        if self.vmode == _lib.VALS_LOAD:
            if vals_in is None or vals_in.numel() != self.n:
                raise ValueError("vals='load' needs a payload tensor of n elements")
            _check_cuda(vals_in, "vals")
        vin = vals_in.data_ptr() if (vals_in is not None and self.vmode == _lib.VALS_LOAD) else None
        if self.graph and self.n > 0 and not eager:
            key = (keys.data_ptr(), vin)
            if self._graph is not None and self._graph_key == key:
                if self._status is not None:
                    self._status.zero_()
                with self._on(stream):  # replay and finish on the caller's stream
                    self._graph.replay()
                self._finish(keys, stream)
                return self.keys_out, self.vals_out
            if self._graph_key != key:  # first call with this input: eager (one-time library setup)
                self._graph, self._graph_key = None, key
                return self._run(keys, vin, stream)
            lib = _lib.load()
            torch.cuda.synchronize(self.device)
            g = torch.cuda.CUDAGraph()
            l0 = lib.isort_launch_count()
            with torch.cuda.graph(g):
                if self._status is not None:
                    self._run_async(keys, vin)
                else:
                    self._run(keys, vin, None)
            self.launches_per_call = int(lib.isort_launch_count() - l0)
            self._graph = g
            if self._status is not None:
                self._status.zero_()
            with self._on(stream):
                g.replay()
            self._finish(keys, stream)
            return self.keys_out, self.vals_out
        return self._run(keys, vin, stream)

    @staticmethod
    def _on(stream):
        import contextlib

        return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()

    def _run_async(self, keys, vin):
        lib = _lib.load()
        s = torch.cuda.current_stream(self.device).cuda_stream
        vout = self.vals_out.data_ptr() if self.vals_out is not None else None
        _lib.check(lib.isort_bucket_sort_u32_async(keys.data_ptr(), self.keys_out.data_ptr(), vin, vout, self.n,
                                                   int(self.range_bound), self.vmode, self.temp.data_ptr(),
                                                   self.temp_bytes, self._status.data_ptr(), s))

    def _finish(self, keys, stream):
        """Bucket graphs: wait for the replay's status, then report / fall back."""
        if self._status is None:
            return
        st = stream or torch.cuda.current_stream(self.device)
        st.synchronize()
        vout = self.vals_out.data_ptr() if self.vals_out is not None else None
        _lib.check(_lib.load().isort_bucket_finish_u32(keys.data_ptr(), self.keys_out.data_ptr(), vout, self.n,
                                                       int(self.range_bound), self.vmode, self.temp.data_ptr(),
                                                       self.temp_bytes, self._status.data_ptr(), st.cuda_stream))

    def _run(self, keys, vin, stream):
        lib = _lib.load()
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        vout = self.vals_out.data_ptr() if self.vals_out is not None else None
        if self.algorithm == RADIX:
            fn = lib.isort_radix_sort_u32 if self.key_bytes == 4 else lib.isort_radix_sort_u64
            rc = fn(keys.data_ptr(), self.keys_out.data_ptr(), vin, vout, self.n, self.vmode,
                    self.temp.data_ptr(), self.temp_bytes, s)
        elif self.range_lo:
            rc = lib.isort_bucket_sort_span_u32(keys.data_ptr(), self.keys_out.data_ptr(), vin, vout, self.n,
                                                self.range_lo, int(self.range_bound), self.vmode,
                                                self.temp.data_ptr(), self.temp_bytes, s)
        else:
            fn = lib.isort_bucket_sort_u32 if self.key_bytes == 4 else lib.isort_bucket_sort_u64
            rc = fn(keys.data_ptr(), self.keys_out.data_ptr(), vin, vout, self.n, int(self.range_bound),
                    self.vmode, self.temp.data_ptr(), self.temp_bytes, s)
        _lib.check(rc)
        return self.keys_out, self.vals_out


def radix_sort(keys: torch.Tensor, vals: torch.Tensor | None = None, iota: bool = False):
    """One-shot device LSD radix sort.  Returns (sorted keys, payload or None)."""
    mode = "load" if vals is not None else ("iota" if iota else None)
    s = Sorter(keys.numel(), _key_bytes(keys), RADIX, mode, device=keys.device)
    k, v = s(keys, vals)
    return k, v


def bucket_sort(keys: torch.Tensor, range_bound: int, vals: torch.Tensor | None = None, iota: bool = False,
                range_lo: int = 0):
    """One-shot device bucket sort over [range_lo, range_bound] (the reference: range_lo = 0)."""
    mode = "load" if vals is not None else ("iota" if iota else None)
    s = Sorter(keys.numel(), _key_bytes(keys), BUCKET, mode, range_bound=range_bound, device=keys.device,
               range_lo=range_lo)
    k, v = s(keys, vals)
    return k, v


def counting_pass(keys: torch.Tensor, base: int, digits: int, digit_index: int, vals: torch.Tensor | None = None,
                  iota: bool = False):
    """One stable device counting pass of u32 keys by digit (key / base^digit_index) mod base
    (counting_sort_by_digit, sort.cpp:77-110).  Returns (keys, payload or None)."""
    _check_cuda(keys, "keys")
    if _key_bytes(keys) != 4:
        raise TypeError("counting_pass: u32 keys")
    n = keys.numel()
    vmode = _lib.VALS_LOAD if vals is not None else (_lib.VALS_IOTA if iota else _lib.VALS_NONE)
    if vals is not None:
        _check_cuda(vals, "vals")
    lib = _lib.load()
    tb = lib.isort_counting_pass_temp_bytes(n)
    temp = torch.empty(max(tb, 1), dtype=torch.uint8, device=keys.device)
    out = torch.empty_like(keys)
    vout = torch.empty(n, dtype=torch.int32, device=keys.device) if vmode != _lib.VALS_NONE else None
    s = torch.cuda.current_stream(keys.device).cuda_stream
    _lib.check(lib.isort_counting_pass_u32(keys.data_ptr(), out.data_ptr(),
                                           vals.data_ptr() if vals is not None else None,
                                           vout.data_ptr() if vout is not None else None, n, int(base), int(digits),
                                           int(digit_index), vmode, temp.data_ptr(), tb, s))
    return out, vout


def is_sorted_u32(keys: torch.Tensor) -> bool:
    import ctypes

    _check_cuda(keys, "keys")
    r = ctypes.c_int(0)
    _lib.check(_lib.load().isort_is_sorted_u32(keys.data_ptr(), keys.numel(), ctypes.byref(r),
                                               torch.cuda.current_stream(keys.device).cuda_stream))
    return bool(r.value)
