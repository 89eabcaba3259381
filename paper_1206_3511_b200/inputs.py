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


def uniform_u32(n: int, seed: int = 42, bits: int = 32, chunk: int = 1 << 24) -> np.ndarray:
    """Keys of generate({case 1, n, M = 2^bits - 1, seed}) as uint32."""
    out = np.empty(n, dtype=np.uint32)
    mask = np.uint64((1 << bits) - 1)
    for s in range(0, n, chunk):
        c = min(chunk, n - s)
        with np.errstate(over="ignore"):
            out[s:s + c] = (_stream(seed, s, c) & mask).astype(np.uint32)
    return out


def mixture_u32(n: int, seed: int = 42, chunk: int = 1 << 22) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32)
    for s in range(0, n, chunk):
        c = min(chunk, n - s)
        i = np.arange(s, s + c, dtype=np.uint64)
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


def config_range_bound(name: str) -> int:
    """Inclusive key bound the bucket sort partitions against, per config."""
    return 1023 if name.lower() == "c3" else (1 << 32) - 1
