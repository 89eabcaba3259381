"""B200 parity tests of the bulk-copy (TMA) one-sweep pass, k_onesweep_t
(radix_onesweep_tma.cuh): u32 sorts of at least 4M keys take it (16,384-key
tiles; 8,192-pair tiles with a payload), so these cases sit right at and above
that size, around its tile boundaries, with the distributions that drive its
special paths (sorted runs -> warp-aggregated rank, one digit -> one run per
tile, two values -> two long runs), and with output arrays that are not
16-byte aligned (the run interiors are staged at the global position modulo one
16-byte block; a payload array on another phase leaves by plain stores).

Reference semantics: the stable counting pass of sort.cpp:77-110, checked bit
for bit against the oracle's stable sort (keys and positions)."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

U32_MAX = (1 << 32) - 1
KS = 4 << 20  # kSmallN: the smallest input that takes the pass
TILE, TILE_V = 16384, 8192
SIZES = [KS, KS + 1, KS + TILE_V - 1, KS + TILE_V + 1, KS + TILE - 1, KS + TILE + 5, KS + 3 * TILE + 4097, 5_000_011]
DISTS = ["uniform", "small_range", "all_equal", "sorted", "reverse", "one_digit", "max_key", "two_values", "runs"]


def _keys(name, n, rng):
    u = lambda: rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)  # noqa: E731
    if name == "uniform":
        return u()
    if name == "small_range":
        return rng.integers(0, 70000, size=n, dtype=np.uint64).astype(np.uint32)  # above the counting pass's range
    if name == "all_equal":
        return np.full(n, 123456789, dtype=np.uint32)
    if name == "sorted":
        k = np.sort(u())
        k[n // 2], k[n // 2 + 1] = k[n // 2 + 1], k[n // 2]  # one inversion: no sorted early-out
        return k
    if name == "reverse":
        k = np.sort(u())[::-1].copy()
        k[n // 3], k[n // 3 + 1] = k[n // 3 + 1], k[n // 3]  # one ascent: no reversal early-out
        return k
    if name == "one_digit":
        return (rng.integers(0, 256, size=n, dtype=np.uint64).astype(np.uint32) << 16) | 0x0A0000BB
    if name == "max_key":
        a = u()
        a[:: max(1, n // 7)] = U32_MAX
        return a
    if name == "two_values":
        return np.where(rng.integers(0, 2, size=n) > 0, U32_MAX, 0).astype(np.uint32)
    if name == "runs":  # sorted runs of 40,000 keys: tiles with few distinct digits in the high passes
        return np.concatenate([np.sort(c) for c in np.array_split(u(), max(1, n // 40000))])
    raise KeyError(name)


def _sort(keys_np, algorithm, payload):
    import torch

    from paper_1206_3511_b200 import device

    t = torch.from_numpy(keys_np.view(np.int32).copy()).cuda()
    s = device.Sorter(keys_np.size, 4, algorithm, payload, range_bound=U32_MAX)
    k, v = s(t)
    torch.cuda.synchronize()
    return k.cpu().numpy().view(np.uint32), (v.cpu().numpy().view(np.uint32) if v is not None else None)


@pytest.mark.parametrize("algorithm", ["radix", "bucket"])
@pytest.mark.parametrize("dist", DISTS)
def test_tma_pass_bit_exact(cuda, oracle, algorithm, dist):
    rng = np.random.default_rng(abs(hash((algorithm, dist))) & 0xFFFF)
    i0 = DISTS.index(dist)
    for j in range(3):  # three of the sizes per distribution (all sizes are covered over the distributions)
        n = SIZES[(i0 + 3 * j) % len(SIZES)]
        k = _keys(dist, n, rng)
        want_k, want_i = oracle.sort_u32(k, with_index=True)
        got_k, _ = _sort(k, algorithm, None)
        assert np.array_equal(got_k, want_k), (algorithm, dist, n, "keys")
        got_k, got_i = _sort(k, algorithm, "iota")
        assert np.array_equal(got_k, want_k), (algorithm, dist, n, "pairs keys")
        assert np.array_equal(got_i, want_i), (algorithm, dist, n, "pairs positions")


@pytest.mark.parametrize("off_k,off_v", [(1, 1), (3, 3), (1, 2), (2, 0), (0, 3)])
def test_tma_pass_unaligned_outputs(cuda, oracle, off_k, off_v):
    """keys_out / vals_out that start 4, 8 or 12 bytes past a 16-byte boundary: the staged
    slot follows the output's phase; a payload array on another phase than the keys
    leaves by plain stores."""
    import torch

    from paper_1206_3511_b200 import _lib

    lib = _lib.load()
    n = KS + TILE + 77
    k = oracle.uniform_u32(n, 11 + off_k * 4 + off_v)
    want_k, want_i = oracle.sort_u32(k, with_index=True)
    kin = torch.from_numpy(k.view(np.int32).copy()).cuda()
    kout = torch.full((n + 8,), -1, dtype=torch.int32, device="cuda")
    vout = torch.full((n + 8,), -1, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    for vals_mode in (0, 2):  # keys only; positions generated on the device
        tb = lib.isort_radix_temp_bytes(n, 4, 1 if vals_mode else 0)
        temp = torch.empty(tb, dtype=torch.uint8, device="cuda")
        kout.fill_(-1)
        vout.fill_(-1)
        _lib.check(lib.isort_radix_sort_u32(kin.data_ptr(), kout.data_ptr() + 4 * off_k, None,
                                            vout.data_ptr() + 4 * off_v if vals_mode else None, n, vals_mode,
                                            temp.data_ptr(), tb, stream))
        torch.cuda.synchronize()
        got = kout.cpu().numpy().view(np.uint32)
        assert np.array_equal(got[off_k:off_k + n], want_k), (off_k, off_v, vals_mode)
        assert np.all(got[:off_k] == U32_MAX) and np.all(got[off_k + n:] == U32_MAX), "wrote outside keys_out"
        if vals_mode:
            gv = vout.cpu().numpy().view(np.uint32)
            assert np.array_equal(gv[off_v:off_v + n], want_i), (off_k, off_v)
            assert np.all(gv[:off_v] == U32_MAX) and np.all(gv[off_v + n:] == U32_MAX), "wrote outside vals_out"


def test_tma_pass_loaded_payload(cuda, oracle):
    """A caller-supplied payload (ISORT_VALS_LOAD) through the pass: values follow their keys stably."""
    import torch

    from paper_1206_3511_b200 import _lib

    lib = _lib.load()
    n = KS + 12345
    k = (oracle.uniform_u32(n, 5) >> 20).astype(np.uint32) << 9  # 4,096 key values above the counting range
    vals = oracle.uniform_u32(n, 6)
    order = np.argsort(k, kind="stable")
    kin = torch.from_numpy(k.view(np.int32).copy()).cuda()
    vin = torch.from_numpy(vals.view(np.int32).copy()).cuda()
    kout, vout = torch.empty_like(kin), torch.empty_like(vin)
    tb = lib.isort_radix_temp_bytes(n, 4, 1)
    temp = torch.empty(tb, dtype=torch.uint8, device="cuda")
    _lib.check(lib.isort_radix_sort_u32(kin.data_ptr(), kout.data_ptr(), vin.data_ptr(), vout.data_ptr(), n, 1,
                                        temp.data_ptr(), tb, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert np.array_equal(kout.cpu().numpy().view(np.uint32), k[order])
    assert np.array_equal(vout.cpu().numpy().view(np.uint32), vals[order])


@pytest.mark.parametrize("n", [KS, KS + 8191, KS + 8193, 5_000_011])
@pytest.mark.parametrize("bits", [64, 40])
def test_tma_pass_u64_keys(cuda, n, bits):
    """u64 keys (keys only) take the pass with 8,192-key tiles and 16-byte blocks of two keys;
    40-bit keys (the reference generator's range) skip the three trivial high passes."""
    import torch

    from paper_1206_3511_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(n % 1000 + bits)
    k = rng.integers(0, 1 << 63, size=n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=n, dtype=np.uint64)
    if bits < 64:
        k >>= np.uint64(64 - bits)
    kin = torch.from_numpy(k.view(np.int64).copy()).cuda()
    for off in (0, 1):  # output on / 8 bytes off a 16-byte boundary
        kout = torch.full((n + 2,), -1, dtype=torch.int64, device="cuda")
        tb = lib.isort_radix_temp_bytes(n, 8, 0)
        temp = torch.empty(tb, dtype=torch.uint8, device="cuda")
        _lib.check(lib.isort_radix_sort_u64(kin.data_ptr(), kout.data_ptr() + 8 * off, None, None, n, 0,
                                            temp.data_ptr(), tb, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        got = kout.cpu().numpy().view(np.uint64)
        assert np.array_equal(got[off:off + n], np.sort(k)), (n, bits, off)
        assert got[off + n] == np.uint64(0xFFFFFFFFFFFFFFFF) and (off == 0 or got[0] == np.uint64(0xFFFFFFFFFFFFFFFF))


@pytest.mark.parametrize("n", [KS + 6143, KS + 6145, 5_000_011])
@pytest.mark.parametrize("off_k,off_v", [(0, 0), (1, 2), (0, 1)])
def test_tma_pass_u64_pairs(cuda, n, off_k, off_v):
    """u64 keys with the position payload (6,144-pair tiles): slots follow the payload array's
    16-byte phase; the key array leaves by bulk copies when its phase agrees modulo two keys
    ((0, 0) and (1, 2)), by plain stores otherwise ((0, 1))."""
    import torch

    from paper_1206_3511_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(n % 977 + 3 * off_k + off_v)
    k = rng.integers(0, 1 << 40, size=n, dtype=np.uint64)  # the reference generator's 40-bit keys, with duplicates
    k[:: 97] = k[0]
    order = np.argsort(k, kind="stable")
    kin = torch.from_numpy(k.view(np.int64).copy()).cuda()
    kout = torch.full((n + 2,), -1, dtype=torch.int64, device="cuda")
    vout = torch.full((n + 4,), -1, dtype=torch.int32, device="cuda")
    tb = lib.isort_radix_temp_bytes(n, 8, 1)
    temp = torch.empty(tb, dtype=torch.uint8, device="cuda")
    _lib.check(lib.isort_radix_sort_u64(kin.data_ptr(), kout.data_ptr() + 8 * off_k, None, vout.data_ptr() + 4 * off_v,
                                        n, 2, temp.data_ptr(), tb, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    got = kout.cpu().numpy().view(np.uint64)
    gv = vout.cpu().numpy().view(np.uint32)
    assert np.array_equal(got[off_k:off_k + n], k[order]), (n, off_k, off_v)
    assert np.array_equal(gv[off_v:off_v + n], order.astype(np.uint32)), (n, off_k, off_v)
    assert np.all(gv[:off_v] == U32_MAX) and np.all(gv[off_v + n:] == U32_MAX), "wrote outside vals_out"
    assert got[off_k + n] == np.uint64(0xFFFFFFFFFFFFFFFF), "wrote outside keys_out"
