"""Operator registry and timing harness, mirroring proj/core/include/intsort/bench.hpp.

``make_sort_fn`` is the reference's plugin point (bench.hpp:44-49,
bench.cpp:55-65): it binds an :class:`AlgorithmId` to a ``SortFn`` closure.  Here
the closures call the B200 engine (paper_1206_3511_b200.intsort).
``time_sort`` follows bench.cpp:67-99: one untimed warm-up (checked), then
``repeats`` timed runs on fresh copies, median and relative spread; an
unsorted output rejects the measurement.
"""
from __future__ import annotations

import enum
import time
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import intsort


class AlgorithmId(enum.Enum):  # bench.hpp:15
    bucket = 0
    radix = 1
    insertion = 2


def algorithm_name(a: AlgorithmId) -> str:  # bench.cpp:30-41
    return a.name


def parse_algorithm(name: str) -> AlgorithmId | None:  # bench.cpp:42-53
    try:
        return AlgorithmId[name]
    except KeyError:
        return None


SortFn = Callable[[np.ndarray], np.ndarray]  # bench.hpp:44


def make_sort_fn(alg: AlgorithmId, range_bound: int, radix_base: int) -> SortFn:  # bench.cpp:55-65
    if alg is AlgorithmId.bucket:
        return lambda seq: intsort.bucket_sort(seq, range_bound)
    if alg is AlgorithmId.radix:
        return lambda seq: intsort.radix_sort_lsd(seq, radix_base)
    if alg is AlgorithmId.insertion:
        return lambda seq: intsort.insertion_sort(seq)
    raise ValueError("make_sort_fn: unknown algorithm")


@dataclass
class TimingStats:  # bench.hpp:53-56
    median_s: float = 0.0
    relative_spread: float = 0.0


def _is_sorted(seq: np.ndarray) -> bool:  # verify.cpp:67-74
    k = seq["key"]
    return bool(np.all(k[:-1] <= k[1:])) if k.size > 1 else True


def time_sort(sort: SortFn, seq: np.ndarray, repeats: int) -> TimingStats:  # bench.cpp:67-99
    if repeats < 3:
        raise ValueError(f"time_sort: repeats must be >= 3, got {repeats}")
    if not _is_sorted(sort(seq)):
        raise RuntimeError("time_sort: warm-up run produced unsorted output")
    durations = []
    for run in range(repeats):
        copy = seq.copy()
        t0 = time.perf_counter()
        out = sort(copy)
        t1 = time.perf_counter()
        if not _is_sorted(out):
            raise RuntimeError(f"time_sort: run {run} produced unsorted output, measurement rejected")
        durations.append(t1 - t0)
    durations.sort()
    c = len(durations)
    med = durations[c // 2] if c % 2 else 0.5 * (durations[c // 2 - 1] + durations[c // 2])
    span = durations[-1] - durations[0]
    return TimingStats(med, span / med if med > 0 else 0.0)
