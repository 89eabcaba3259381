"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference's generator (proj/core/src/generator.cpp) draws keys with
SplitMix64 (rng.hpp:13-47).  For a power-of-two bound 2^k, ``below`` never
rejects (2^64 mod 2^k = 0, rng.hpp:33-38), so key i of ``generate({case 1,
n, M = 2^k - 1, seed})`` is ``mix(seed + (i+1)*gamma) & (2^k - 1)``: a
counter-based stream that numpy evaluates vectorised and bit-identically
(tests/test_inputs.py pins it against the oracle restatement).

    C1  n=1e6  u32 uniform [0, 2^32)           generate(case 1, M=2^32-1, seed 42)
    C2  n=1e8  u32 uniform [0, 2^32)           same, n=1e8
    C3  n=1e8  u32 uniform [0, 1024)           generate(case 1, M=1023, seed 42)
    C4a n=1e8  C2 sorted ascending             generate(case 2, M=2^32-1, seed 42)
    C4b        C4a reversed (harness addition)
    C5  n=1e9  mixture: 50% U[0,2^32), 50% N(2^31, 2^24) clamped (harness addition,
               SURVEY.md §8d): component = top bit of x_{3i}; uniform = low 32 bits
               of x_{3i+1}; normal = Box-Muller on x_{3i+1}, x_{3i+2}.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def mix64(z: np.ndarray) -> np.ndarray:
    """SplitMix64 output function (rng.hpp:19-22), vectorised, wrapping."""
    z = (z ^ (z >> np.uint64(30))) * M1
    z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def _stream(seed: int, start: int, count: int, step: int = 1, offset: int = 1) -> np.ndarray:
    """x_j = mix(seed + (j + offset) * gamma) for j = start, start+step, ..."""
    j = np.arange(start, start + count * step, step, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(np.uint64(seed) + (j + np.uint64(offset)) * GAMMA)


def uniform_u32(n: int, seed: int = 42, bits: int = 32, chunk: int = 1 << 24, start: int = 0) -> np.ndarray:
    """Keys start .. start+n-1 of generate({case 1, M = 2^bits - 1, seed}) as uint32
    (the stream is counter-based: a shard is generated without the keys before it)."""
    out = np.empty(n, dtype=np.uint32)
    mask = np.uint64((1 << bits) - 1)
    for s in range(0, n, chunk):
        c = min(chunk, n - s)
        with np.errstate(over="ignore"):
            out[s:s + c] = (_stream(seed, start + s, c) & mask).astype(np.uint32)
    return out


def mixture_u32(n: int, seed: int = 42, chunk: int = 1 << 22, start: int = 0) -> np.ndarray:
    """Keys start .. start+n-1 of the config-5 mixture (counter-based, like uniform_u32)."""
    out = np.empty(n, dtype=np.uint32)
    for s in range(0, n, chunk):
        c = min(chunk, n - s)
        i = np.arange(start + s, start + s + c, dtype=np.uint64)
        with np.errstate(over="ignore"):
            x0 = mix64(np.uint64(seed) + (np.uint64(3) * i + np.uint64(1)) * GAMMA)
            x1 = mix64(np.uint64(seed) + (np.uint64(3) * i + np.uint64(2)) * GAMMA)
            x2 = mix64(np.uint64(seed) + (np.uint64(3) * i + np.uint64(3)) * GAMMA)
        normal = (x0 >> np.uint64(63)) != 0
        u1 = 1.0 - (x1 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        u2 = (x2 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
        v = np.clip(np.floor(2147483648.0 + 16777216.0 * z + 0.5), 0, 4294967295.0).astype(np.uint64)  # llround
        out[s:s + c] = np.where(normal, v, x1 & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    return out


def config_keys(name: str, n: int | None = None, seed: int = 42) -> np.ndarray:
    """Keys (uint32) of a BASELINE configuration by name: c1, c2, c3, c4a, c4b, c5."""
    name = name.lower()
    if name == "c5" and (n or 10**9) >= (1 << 24):
        return mixture_u32_parallel(n or 10**9, seed)
    if name in ("c1", "c2"):
        return uniform_u32(n or (10**6 if name == "c1" else 10**8), seed)
    if name == "c3":
        return uniform_u32(n or 10**8, seed, bits=10)
    if name in ("c4a", "c4b"):
        k = np.sort(uniform_u32(n or 10**8, seed))
        return k if name == "c4a" else k[::-1].copy()
    if name == "c5":
        return mixture_u32(n or 10**9, seed)
    raise KeyError(name)


def mixture_u32_parallel(n: int, seed: int = 42, start: int = 0, threads: int | None = None) -> np.ndarray:
    """mixture_u32 over host threads (numpy drops the GIL in its kernels): the same
    values, each thread filling its own index range."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    out = np.empty(n, dtype=np.uint32)
    threads = threads or min(32, os.cpu_count() or 1)
    step = max(1 << 22, (n + threads - 1) // threads)

    def part(s):
        c = min(step, n - s)
        out[s:s + c] = mixture_u32(c, seed, start=start + s)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(part, range(0, n, step)))
    return out


def config_shard(name: str, n_total: int, rank: int, world: int, seed: int = 42) -> np.ndarray:
    """Rank `rank`'s positional shard [r*n/G, (r+1)*n/G) of a configuration's
    n_total keys: the G shards concatenated are exactly config_keys(name, n_total)."""
    lo, hi = n_total * rank // world, n_total * (rank + 1) // world
    name = name.lower()
    if name in ("c1", "c2"):
        return uniform_u32(hi - lo, seed, start=lo)
    if name == "c3":
        return uniform_u32(hi - lo, seed, bits=10, start=lo)
    if name == "c5":
        return mixture_u32_parallel(hi - lo, seed, start=lo)
    return config_keys(name, n_total, seed)[lo:hi].copy()


def config_range_bound(name: str) -> int:
    """Inclusive key bound the bucket sort partitions against, per config."""
    return 1023 if name.lower() == "c3" else (1 << 32) - 1


# ------------------------------------------------- the reference's six input cases
# generate() (generator.cpp:112-147) over SplitMix64::below (rng.hpp:25-38), exact:
# x_k = mix(seed + (k+1)*gamma) is counter-based, and a rejected draw only skips
# one x, so a batch of draws = the accepted values of a slightly longer batch.
_U64MAX = (1 << 64) - 1


class _Stream:
    def __init__(self, seed: int):
        self.seed, self.ctr = seed, 0

    def raw(self, m: int) -> np.ndarray:
        out = _stream(self.seed, self.ctr, m, offset=1)
        self.ctr += m
        return out

    def below(self, bound: int, m: int) -> np.ndarray:
        """m draws of below(bound) (the same bound)."""
        if bound <= 0:
            raise ValueError("SplitMix64::below: bound must be >= 1")
        lim = np.uint64(_U64MAX - ((1 << 64) - bound) % bound)
        got, parts = 0, []
        while got < m:
            want = m - got
            xs = _stream(self.seed, self.ctr, want + 8, offset=1)
            ok = np.flatnonzero(xs <= lim)[:want]
            take = xs[ok]
            self.ctr += int(ok[-1]) + 1 if ok.size else want + 8
            parts.append(take % np.uint64(bound))
            got += take.size
        return np.concatenate(parts) if parts else np.empty(0, dtype=np.uint64)

    def below_each(self, bounds: np.ndarray) -> np.ndarray:
        """One draw per element, bound bounds[i] (varying), in order."""
        out = np.empty(bounds.size, dtype=np.uint64)
        i = 0
        b64 = bounds.astype(np.uint64)
        while i < bounds.size:
            rest = b64[i:]
            xs = _stream(self.seed, self.ctr, rest.size, offset=1)
            with np.errstate(over="ignore"):
                lim = np.uint64(_U64MAX) - ((np.uint64(0) - rest) % rest)
            bad = np.flatnonzero(xs > lim)
            r = int(bad[0]) if bad.size else rest.size
            out[i:i + r] = xs[:r] % rest[:r]
            self.ctr += r + (1 if bad.size else 0)  # the rejected x is skipped, its bound redrawn
            i += r
        return out


def _mulmod(j: np.ndarray, s: int, m: int) -> np.ndarray:
    """(j * s) mod m without 128-bit products: j < 2^27, s, m < 2^41."""
    jl = j & np.uint64((1 << 20) - 1)
    jh = j >> np.uint64(20)
    a = np.uint64(((1 << 20) * s) % m)
    return ((jh * a) % np.uint64(m) + (jl * np.uint64(s)) % np.uint64(m)) % np.uint64(m)


def default_range_bound(case_id: int) -> int:  # generator.cpp:71-80
    return {4: 10_000, 5: 100_000_000}.get(case_id, 1_000_000)


def generate_case(case_id: int, n: int, range_bound: int | None = None, seed: int = 0,
                  repeated_value: int | None = None, sorted_fraction: float = 0.95) -> np.ndarray:
    """Keys (uint64) of the reference's generate(InputSpec) -- exact for all six
    cases (tests/test_inputs.py pins it against the reference).  Cases 3 and 6
    end in sequential swap loops and are meant for n up to ~10^7."""
    import math

    if case_id < 1 or case_id > 6:
        raise ValueError("InputSpec: case_id must be in 1..6")
    bound = default_range_bound(case_id) if range_bound is None else int(range_bound)
    if bound > (1 << 40):
        raise ValueError("InputSpec: range_bound exceeds 2^40")
    if not 0.0 <= sorted_fraction <= 1.0:
        raise ValueError("InputSpec: sorted_fraction must be in [0, 1]")
    rng = _Stream(seed)
    if case_id in (1, 4, 5):
        return rng.below(bound + 1, n)
    if case_id in (2, 3):
        keys = np.sort(rng.below(bound + 1, n))
        if case_id == 3:
            swaps = int((1.0 - sorted_fraction) * float(n))
            ab = rng.below(n, 2 * swaps) if swaps else np.empty(0, dtype=np.uint64)
            k = keys.tolist()
            for a, b in zip(ab[0::2].tolist(), ab[1::2].tolist()):
                k[a], k[b] = k[b], k[a]
            keys = np.array(k, dtype=np.uint64)
        return keys
    # case 6: ceil(n/3) copies of the repeated value + distinct fillers on a coprime walk, shuffled
    rep = bound // 2 if repeated_value is None else int(repeated_value)
    if rep > bound:
        raise ValueError("InputSpec: repeated_value exceeds range_bound")
    if (2 * n + 2) // 3 > bound:
        raise ValueError(f"InputSpec: case 6 infeasible, ceil(2n/3) = {(2 * n + 2) // 3} exceeds range_bound {bound} "
                         "(not enough distinct values)")
    dup = (n + 2) // 3
    distinct = n - dup
    m = bound + 1
    keys = np.full(n, rep, dtype=np.uint64)
    if distinct > 0:
        while True:
            stride = int(rng.below(m, 1)[0])
            if stride != 0 and math.gcd(stride, m) == 1:
                break
        v = int(rng.below(m, 1)[0])
        walk = (np.uint64(v) + _mulmod(np.arange(distinct + 1, dtype=np.uint64), stride, m)) % np.uint64(m)
        walk = walk[walk != np.uint64(rep)][:distinct]
        keys[dup:] = walk
    js = rng.below_each(np.arange(n, 1, -1, dtype=np.uint64))  # Fisher-Yates, i = n .. 2
    k = keys.tolist()
    for i, j in zip(range(n, 1, -1), js.tolist()):
        k[i - 1], k[j] = k[j], k[i - 1]
    return np.array(k, dtype=np.uint64)
