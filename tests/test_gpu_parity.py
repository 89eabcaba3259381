"""GPU parity: the sm_100a engine against the oracle and the reference's golden
vectors.  Bit-exact for keys and payload (positions) -- a stable sort has one
correct output.  Run with ``-m gpu`` on a B200."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

import paper_1206_3511_b200 as isort
from oracle.binding import RECORD_DTYPE

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
U32_MAX = (1 << 32) - 1
# one-sweep geometry: chunk = 512 threads x IPT keys, tile = 2 chunks
# (keys-only IPT 24: 12288 / 24576; with payload IPT 12: 6144 / 12288; below 4M keys
# one chunk per tile: 8192 keys-only, 6144 with payload)
TILE = 24576
BOUNDARIES = [4095, 4096, 4097, 6143, 6144, 6145, 8191, 8192, 8193, 12287, 12288, 12289, 16384, 24575, 24576, 24577,
              2 * 24576 + 17, 3 * 12288 + 5]


def recs(keys):
    a = np.empty(len(keys), dtype=RECORD_DTYPE)
    a["key"] = np.asarray(keys, dtype=np.uint64)
    a["tag"] = np.arange(len(keys), dtype=np.uint64)
    return a


def dev_sort(keys_np: np.ndarray, algorithm="radix", payload="iota", range_bound=None):
    import torch

    from paper_1206_3511_b200 import device

    kb = keys_np.dtype.itemsize
    t = torch.from_numpy(keys_np.view(np.int32 if kb == 4 else np.int64).copy()).cuda()
    s = device.Sorter(keys_np.size, kb, algorithm, payload, range_bound=range_bound)
    k, v = s(t)
    torch.cuda.synchronize()
    ko = k.cpu().numpy().view(keys_np.dtype)
    vo = v.cpu().numpy().view(np.uint32) if v is not None else None
    return ko, vo


# ------------------------------------------------------- golden vectors (records API)
@pytest.fixture(scope="module")
def golden():
    z = np.load(os.path.join(GOLDEN, "reference_vectors.npz"))
    with open(os.path.join(GOLDEN, "reference_vectors.json")) as f:
        meta = json.load(f)
    return z, meta


def test_records_radix_matches_reference_vectors(cuda, golden):
    z, meta = golden
    for i, sp in enumerate(meta):
        s = recs(z[f"in_{i}"])
        out10 = isort.radix_sort_lsd(s, 10)
        assert np.array_equal(out10["tag"], z[f"radix10_{i}"]), sp
        assert np.array_equal(out10["key"], s["key"][z[f"radix10_{i}"]]), sp
        assert np.array_equal(isort.radix_sort_lsd(s, 256)["tag"], z[f"radix256_{i}"]), sp


def test_records_bucket_matches_reference_vectors(cuda, golden):
    z, meta = golden
    for i, sp in enumerate(meta):
        s = recs(z[f"in_{i}"])
        out = isort.bucket_sort(s, sp["bound"])
        assert np.array_equal(out["tag"], z[f"bucket_{i}"]), sp


def test_records_plan_and_counting_pass_match_reference(cuda, golden):
    z, meta = golden
    for i, sp in enumerate(meta):
        s = recs(z[f"in_{i}"])
        assert isort.build_radix_plan(s, 10).digits == sp["digits10"]
        assert isort.build_radix_plan(s, 256).digits == sp["digits256"]
        if sp["n"]:
            d = sp["digits10"]
            out = isort.counting_sort_by_digit(s, isort.RadixPlan(10, d), d - 1)
            assert np.array_equal(out["tag"], z[f"count_top_{i}"]), sp


def test_device_bucket_index_matches_reference(cuda, golden):
    z, _ = golden
    bi = z["bucket_index"]
    # group by (count, bound) is unnecessary: one call per sample keeps the test simple
    for key, count, bound, want in bi[:300].tolist():
        assert isort.bucket_index(int(key), int(count), int(bound)) == int(want)
    with pytest.raises(isort.InvalidArgument, match="exceeds range bound"):
        isort.bucket_index(1000, 10, 999)
    with pytest.raises(isort.InvalidArgument):
        isort.bucket_index(0, 0, 999)


# ------------------------------------------------------- device API vs oracle
SIZES = [1, 2, 31, 32, 33, 1000, *BOUNDARIES, 100_000, 1_000_003]


def _dist(name, n, rng):
    if name == "uniform":
        return rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    if name == "small_range":
        return rng.integers(0, 1024, size=n, dtype=np.uint64).astype(np.uint32)
    if name == "all_equal":
        return np.full(n, 123456789, dtype=np.uint32)
    if name == "sorted":
        return np.sort(rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32))
    if name == "reverse":
        return np.sort(rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32))[::-1].copy()
    if name == "one_digit":  # only digit 2 varies
        return (rng.integers(0, 256, size=n, dtype=np.uint64).astype(np.uint32) << 16) | 0x0A0000BB
    if name == "max_key":
        a = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
        a[:: max(1, n // 7)] = U32_MAX
        return a
    if name == "two_values":
        return np.where(rng.integers(0, 2, size=n) > 0, U32_MAX, 0).astype(np.uint32)
    raise KeyError(name)


DISTS = ["uniform", "small_range", "all_equal", "sorted", "reverse", "one_digit", "max_key", "two_values"]


@pytest.mark.parametrize("algorithm", ["radix", "bucket"])
@pytest.mark.parametrize("dist", DISTS)
def test_device_u32_pairs_bit_exact(cuda, oracle, algorithm, dist):
    rng = np.random.default_rng(hash((algorithm, dist)) & 0xFFFF)
    for n in SIZES:
        k = _dist(dist, n, rng)
        want_k, want_i = oracle.sort_u32(k, with_index=True)
        got_k, got_i = dev_sort(k, algorithm, "iota", range_bound=U32_MAX)
        assert np.array_equal(got_k, want_k), (algorithm, dist, n)
        assert np.array_equal(got_i, want_i), (algorithm, dist, n)


@pytest.mark.parametrize("algorithm", ["radix", "bucket"])
def test_device_u32_keys_only(cuda, oracle, algorithm):
    rng = np.random.default_rng(5)
    for dist in DISTS:
        for n in (0, 1, 5000, TILE * 3 + 1, 2_000_000):
            k = _dist(dist, n, rng) if n else np.zeros(0, dtype=np.uint32)
            got, _ = dev_sort(k, algorithm, None, range_bound=U32_MAX)
            assert np.array_equal(got, np.sort(k)), (algorithm, dist, n)


def test_device_u32_loaded_payload(cuda, oracle):
    import torch

    from paper_1206_3511_b200 import device

    rng = np.random.default_rng(11)
    n = 300_001
    k = rng.integers(0, 1 << 20, size=n, dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    order = np.argsort(k, kind="stable")
    for alg in ("radix", "bucket"):
        s = device.Sorter(n, 4, alg, "load", range_bound=(1 << 20) - 1)
        ko, vo = s(torch.from_numpy(k.view(np.int32)).cuda(), torch.from_numpy(v.view(np.int32)).cuda())
        assert np.array_equal(ko.cpu().numpy().view(np.uint32), k[order])
        assert np.array_equal(vo.cpu().numpy().view(np.uint32), v[order])


@pytest.mark.parametrize("algorithm", ["radix", "bucket"])
def test_device_u64_pairs(cuda, algorithm):
    rng = np.random.default_rng(17)
    for n, hi in [(1, 40), (9999, 40), (200_001, 40), (200_001, 64), (50_000, 8)]:
        k = rng.integers(0, 1 << min(hi, 63), size=n, dtype=np.uint64)
        if hi == 64:
            k |= rng.integers(0, 2, size=n, dtype=np.uint64) << np.uint64(63)
        want = np.argsort(k, kind="stable").astype(np.uint32)
        got_k, got_i = dev_sort(k, algorithm, "iota", range_bound=(1 << 64) - 1)
        assert np.array_equal(got_i, want), (algorithm, n, hi)
        assert np.array_equal(got_k, k[want])


# ------------------------------------------------------- bucket-specific semantics
@pytest.mark.parametrize("bound", [U32_MAX, 1023, 1 << 40, 10**8, 999_999, (1 << 64) - 1, 3 * 10**9 + 7])
def test_bucket_range_bounds(cuda, oracle, bound):
    rng = np.random.default_rng(bound & 0xFFFF)
    hi = min(bound, U32_MAX)
    for n in (10, 4097, 123_457):
        k = rng.integers(0, hi + 1, size=n, dtype=np.uint64).astype(np.uint32)
        want_k, want_i = oracle.sort_u32(k, with_index=True)
        got_k, got_i = dev_sort(k, "bucket", "iota", range_bound=bound)
        assert np.array_equal(got_i, want_i), (bound, n)


def test_bucket_range_error_names_first_offending_key(cuda):
    s = recs([5, 3, 11, 2, 12])
    with pytest.raises(isort.InvalidArgument, match=r"bucket_index: key 11 exceeds range bound 10 "
                                                    r"\(sequence/spec mismatch\)"):
        isort.bucket_sort(s, 10)
    from paper_1206_3511_b200 import _lib

    assert _lib.load().isort_last_bad_index() == 2
    with pytest.raises(isort.InvalidArgument):
        isort.bucket_sort(recs([11]), 10)  # test_sort.cpp:192


def test_bucket_oversized_super_buckets(cuda, oracle):
    """All keys in one bucket (M far above the keys): one oversized, non-constant
    super-bucket -> radix fallback; and constant oversized super-buckets (heavy
    duplicates, config 3 shape) that must keep arrival order."""
    rng = np.random.default_rng(3)
    n = 1_000_000
    small = rng.integers(0, 1024, size=n, dtype=np.uint64).astype(np.uint32)
    for bound in (U32_MAX, 1023):
        want_k, want_i = oracle.sort_u32(small, with_index=True)
        got_k, got_i = dev_sort(small, "bucket", "iota", range_bound=bound)
        assert np.array_equal(got_i, want_i), bound
    mix = oracle.mixture_u32(2_000_000, 42)
    want_k, want_i = oracle.sort_u32(mix, with_index=True)
    got_k, got_i = dev_sort(mix, "bucket", "iota", range_bound=U32_MAX)
    assert np.array_equal(got_i, want_i)


@pytest.mark.parametrize("n", [1000, 4099, 1_000_003, 5_000_001])
def test_single_inversion_defeats_sorted_early_out(cuda, n):
    """The histogram kernel's sortedness check (the sorted-input early-out) must see
    one adjacent inversion anywhere: inside a 4-key group, across lanes, across a
    warp's 512-byte blocks and steps, and in the scalar tail."""
    base = np.arange(n, dtype=np.uint64) * 3 + 7
    for p in sorted(q for q in {0, 2, 3, 4, 127, 128, 511, 512, 2047, 2048, n // 2, n - 5, n - 4, n - 3, n - 2}
                    if q + 1 < n):
        k = base.copy()
        k[p], k[p + 1] = k[p + 1], k[p]
        k = k.astype(np.uint32)
        want = np.sort(k)
        for alg in ("radix", "bucket"):
            got, _ = dev_sort(k, alg, None, range_bound=(1 << 32) - 1 if alg == "bucket" else None)
            assert np.array_equal(got, want), (n, p, alg)


@pytest.mark.parametrize("base,digits,idx", [(10, 10, 0), (10, 10, 3), (10, 10, 9), (256, 4, 1), (2, 32, 31),
                                              (1000, 4, 2), (65536, 2, 1), ((1 << 20) + 5, 2, 1), (7, 12, 11)])
def test_device_counting_pass(cuda, oracle, base, digits, idx):
    """isort_counting_pass_u32 against the oracle's counting_sort_by_digit (sort.cpp:77-110)."""
    import torch

    from paper_1206_3511_b200 import device

    rng = np.random.default_rng(base % 9973 + idx)
    for n in (1, 1000, 100_003):
        k = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
        want = oracle.counting_sort_by_digit(recs(k), base, digits, idx)
        t = torch.from_numpy(k.view(np.int32).copy()).cuda()
        ko, vo = device.counting_pass(t, base, digits, idx, iota=True)
        assert np.array_equal(ko.cpu().numpy().view(np.uint32), want["key"].astype(np.uint32)), (base, idx, n)
        assert np.array_equal(vo.cpu().numpy().view(np.uint32), want["tag"].astype(np.uint32)), (base, idx, n)
        v = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
        ko, vo = device.counting_pass(t, base, digits, idx, vals=torch.from_numpy(v.view(np.int32)).cuda())
        assert np.array_equal(vo.cpu().numpy().view(np.uint32), v[want["tag"].astype(np.int64)]), (base, idx, n)


def test_device_counting_pass_errors(cuda):
    import torch

    from paper_1206_3511_b200 import device

    t = torch.zeros(4, dtype=torch.int32, device="cuda")
    with pytest.raises(isort.InvalidArgument, match="base must be >= 2"):
        device.counting_pass(t, 1, 3, 0)
    with pytest.raises(isort.InvalidArgument, match="digit_index 3 out of range for a 3-digit plan"):
        device.counting_pass(t, 10, 3, 3)


@pytest.mark.parametrize("lo,hi", [(0, U32_MAX), (7 << 29, U32_MAX), (1 << 31, (1 << 31) + (1 << 24)),
                                   (12345, 12345 + 1023), (1000, 1000), (5, U32_MAX - 1), (3, 10**8)])
def test_bucket_span_sort(cuda, oracle, lo, hi):
    """isort_bucket_sort_span_u32 (the multi-GPU local step): n buckets over
    [lo, hi].  Any stable sort of the keys is the one correct output."""
    import torch

    from paper_1206_3511_b200 import device

    rng = np.random.default_rng(lo ^ (hi & 0xFFFF))
    for n in (10, 4097, 1_000_003):
        u = rng.integers(lo, hi + 1, size=n, dtype=np.uint64)
        c = np.clip(np.rint((lo + hi) / 2 + (hi - lo) / 64 * rng.standard_normal(n)), lo, hi).astype(np.uint64)
        k = np.where(rng.integers(0, 2, size=n) > 0, u, c).astype(np.uint32)
        want_k, want_i = oracle.sort_u32(k, with_index=True)
        t = torch.from_numpy(k.view(np.int32).copy()).cuda()
        got_k, got_v = device.bucket_sort(t, hi, iota=True, range_lo=lo)
        assert np.array_equal(got_k.cpu().numpy().view(np.uint32), want_k), (lo, hi, n)
        assert np.array_equal(got_v.cpu().numpy().view(np.uint32), want_i), (lo, hi, n)
        got_k, _ = device.bucket_sort(t, hi, range_lo=lo)  # keys only
        assert np.array_equal(got_k.cpu().numpy().view(np.uint32), want_k), (lo, hi, n)


@pytest.mark.parametrize("lo,hi", [(7 << 29, U32_MAX), (1 << 30, (3 << 30) - 1), (12345, 12345 + (1 << 24) - 1),
                                   (1000, 10**9 + 999), (0, 3 * 10**9)])
def test_bucket_span_uniform_takes_no_fallback(cuda, lo, hi):
    """Uniform keys over [lo, hi] spread ~1 key per bucket: every super-bucket fits a
    stage, so the oversized-span radix fallback must not run (it did, silently, while
    the reciprocal of power-of-two spans was missing -- correct output, 30x slower)."""
    import ctypes

    import torch

    from paper_1206_3511_b200 import _lib, device

    lib = _lib.load()
    n = 1_000_003
    k = np.random.default_rng(lo % 997).integers(lo, hi + 1, size=n, dtype=np.uint64).astype(np.uint32)
    t = torch.from_numpy(k.view(np.int32).copy()).cuda()
    s = device.Sorter(n, 4, "bucket", None, range_bound=hi, range_lo=lo)
    s(t)
    torch.cuda.synchronize()
    assert lib.isort_profile_begin() == 0
    s(t)
    torch.cuda.synchronize()
    ms = (ctypes.c_float * 512)()
    names = ctypes.create_string_buffer(512 * 16)
    cnt, na = ctypes.c_int(0), ctypes.c_int(0)
    assert lib.isort_profile_end(ms, names, 16, 512, ctypes.byref(cnt), ctypes.byref(na)) == 0
    phases = [names.raw[i * 16:(i + 1) * 16].split(b"\0")[0].decode() for i in range(cnt.value)]
    assert "segments" in phases and "fallback" not in phases, phases
    assert np.array_equal(s.keys_out.cpu().numpy().view(np.uint32), np.sort(k))


def test_bucket_span_errors(cuda):
    import torch

    from paper_1206_3511_b200 import _lib, device

    t = torch.from_numpy(np.array([500, 600, 499, 700], dtype=np.uint32).view(np.int32)).cuda()
    with pytest.raises(isort.InvalidArgument, match="key 499 below range base 500"):
        device.bucket_sort(t, 1000, range_lo=500)
    assert _lib.load().isort_last_bad_index() == 2
    with pytest.raises(isort.InvalidArgument, match="exceeds range bound 650"):
        device.bucket_sort(torch.from_numpy(np.array([500, 651], dtype=np.uint32).view(np.int32)).cuda(), 650,
                           range_lo=400)
    with pytest.raises(isort.InvalidArgument, match="range base 700 above range bound 600"):
        device.bucket_sort(t, 600, range_lo=700)


@pytest.mark.parametrize("n", [5000, 8191, 8192, 8193, 20_000, 100_003, 1_000_003])
def test_bucket_segment_kernel_paths(cuda, oracle, n):
    """The segment kernel's in-stage shapes: stages of many small super-buckets
    (narrow keys), duplicates inside a bucket (triples), stages cut inside a
    super-bucket and tight clusters next to empty stretches (clusters: oversized
    super-buckets, constant or re-sorted by the radix fallback)."""
    rng = np.random.default_rng(n)
    cases = {
        "narrow": rng.integers(0, 1 << 20, size=n, dtype=np.uint64).astype(np.uint32),
        "triples": np.repeat(rng.integers(0, 1 << 32, size=(n + 2) // 3, dtype=np.uint64), 3)[:n],
        "clusters": (rng.integers(0, 50, size=n, dtype=np.uint64) * (1 << 26)
                     + rng.integers(0, 1 << 12, size=n, dtype=np.uint64)),
    }
    cases["triples"] = rng.permutation(cases["triples"]).astype(np.uint32)
    cases["clusters"] = cases["clusters"].astype(np.uint32)
    for name, k in cases.items():
        want_k, want_i = oracle.sort_u32(k, with_index=True)
        got_k, got_i = dev_sort(k, "bucket", "iota", range_bound=U32_MAX)
        assert np.array_equal(got_k, want_k), (name, n)
        assert np.array_equal(got_i, want_i), (name, n)


# ------------------------------------------------------- config-shaped checksums (10^6)
def test_config_shaped_checksums_match_reference(cuda, oracle):
    with open(os.path.join(GOLDEN, "reference_checksums.json")) as f:
        checks = json.load(f)
    n = 1_000_000
    inputs = {
        "u32_uniform": oracle.generate(1, n, U32_MAX, 42),
        "u32_small_range_1023": oracle.generate(1, n, 1023, 42),
        "u32_sorted": oracle.generate(2, n, U32_MAX, 42),
    }
    rev = inputs["u32_sorted"][::-1].copy()
    rev["tag"] = np.arange(n, dtype=np.uint64)
    inputs["u32_reverse"] = rev
    inputs["u32_mixture"] = recs(oracle.mixture_u32(n, 42))
    for name, seq in inputs.items():
        c = checks[name]
        assert hashlib.sha256(seq["key"].astype(np.uint32).tobytes()).hexdigest() == c["input_sha256"], name
        for out in (isort.radix_sort_lsd(seq, 256), isort.radix_sort_lsd(seq, 10), isort.bucket_sort(seq, U32_MAX)):
            assert hashlib.sha256(out.tobytes()).hexdigest() == c["sorted_records_sha256"], name


# ------------------------------------------------------- BASELINE-size properties (10^8)
def test_full_size_radix_and_bucket_10e8(cuda, oracle):
    n = 100_000_000
    k = oracle.uniform_u32(n, 42)
    want_k, want_i = oracle.sort_u32(k, with_index=True)
    for alg in ("radix", "bucket"):
        got_k, got_i = dev_sort(k, alg, "iota", range_bound=U32_MAX)
        assert np.array_equal(got_k, want_k), alg
        assert np.array_equal(got_i, want_i), alg
        got_k, _ = dev_sort(k, alg, None, range_bound=U32_MAX)
        assert np.array_equal(got_k, want_k), alg


# ------------------------------------------------------- key-range partition kernel (multi-GPU step 3)
@pytest.mark.parametrize("parts", [2, 3, 8])
def test_partition_kernel_is_stable_grouping(cuda, parts):
    import torch

    from paper_1206_3511_b200.partition import CudaOps

    rng = np.random.default_rng(parts)
    ops = CudaOps(torch.device("cuda:0"))
    for n in (1, 1000, TILE * 5 + 3, 3_000_000):
        k = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
        spl = sorted(int(x) for x in rng.integers(0, 1 << 32, size=parts - 1, dtype=np.uint64))
        v = np.arange(n, dtype=np.int32)
        tk = torch.from_numpy(k.view(np.int32)).cuda()
        tv = torch.from_numpy(v).cuda()
        ok, ov, cnt = ops.partition(tk, tv, spl, parts)
        dest = np.searchsorted(np.array(spl, dtype=np.uint64), k.astype(np.uint64), side="right")
        order = np.argsort(dest, kind="stable")
        assert np.array_equal(cnt.cpu().numpy(), np.bincount(dest, minlength=parts)), (parts, n)
        assert np.array_equal(ok.cpu().numpy().view(np.uint32), k[order]), (parts, n)
        assert np.array_equal(ov.cpu().numpy(), v[order]), (parts, n)


@pytest.mark.parametrize("parts,n_extra,payload", [(2, 0, True), (5, 0, True), (8, 0, True),
                                                   (3, 4_000_000, True), (4, 4_000_000, False)])
def test_fused_partition_scatter_protocol(cuda, oracle, parts, n_extra, payload):
    """The fused exchange's kernels and address arithmetic on one GPU: `parts`
    simulated ranks run one after another (no kernel waits on another).  Each
    counts its shard, the count matrix gives every run's slot, and the partition
    pass stores each run straight into the destination's receive buffer; the
    destinations' stable local sorts concatenate to the global stable sort."""
    import torch

    from paper_1206_3511_b200 import device
    from paper_1206_3511_b200.partition import CudaOps, fused_destinations, recv_totals

    rng = np.random.default_rng(100 + parts)
    n = 2_500_000 + parts * 7919 + n_extra  # n_extra: past the small-n tile shape
    keys = oracle.mixture_u32(n, 40 + parts)
    pos = np.arange(n, dtype=np.int32)
    shards = np.array_split(np.arange(n), parts)
    spl = sorted(int(x) for x in np.quantile(keys[rng.integers(0, n, 4096)], np.arange(1, parts) / parts))
    ops = [CudaOps(torch.device("cuda:0")) for _ in range(parts)]
    tk = [torch.from_numpy(keys[sh].view(np.int32)).cuda() for sh in shards]
    tv = [torch.from_numpy(pos[sh]).cuda() for sh in shards]
    matrix = [[int(c) for c in ops[r].partition_counts(tk[r], spl, parts).tolist()] for r in range(parts)]
    totals = recv_totals(matrix)
    assert sum(totals) == n
    rk = [torch.full((t + 3,), -1, dtype=torch.int32, device="cuda") for t in totals]  # + guard words
    rv = [torch.full((t + 3,), -1, dtype=torch.int32, device="cuda") for t in totals]
    kb, vb = [t.data_ptr() for t in rk], [t.data_ptr() for t in rv]
    for r in range(parts):
        ops[r].partition_scatter(tk[r], tv[r] if payload else None, spl, parts,
                                 fused_destinations(matrix, r, kb, 4),
                                 fused_destinations(matrix, r, vb, 4) if payload else None)
    torch.cuda.synchronize()
    got_k, got_v = [], []
    for d in range(parts):
        assert (rk[d][totals[d]:] == -1).all(), "store past the slot"
        if payload:
            assert (rv[d][totals[d]:] == -1).all(), "payload store past the slot"
            k, v = device.radix_sort(rk[d][: totals[d]].contiguous(), vals=rv[d][: totals[d]].contiguous())
            got_v.append(v.cpu().numpy())
        else:
            k, _ = device.radix_sort(rk[d][: totals[d]].contiguous())
        got_k.append(k.cpu().numpy().view(np.uint32))
    want_k, want_i = oracle.sort_u32(keys, with_index=True)
    assert np.array_equal(np.concatenate(got_k), want_k)
    if payload:
        assert np.array_equal(np.concatenate(got_v).astype(np.uint32), want_i)


@pytest.mark.parametrize("n", [1000, 1_000_000, 5_000_003])
def test_radix_cuda_graph_replay(cuda, oracle, n):
    """Sorter(graph=True): eager first call, then capture, then replays that read
    the (same) input buffer afresh -- bit-exact every time."""
    import torch

    from paper_1206_3511_b200 import device

    rng = np.random.default_rng(n)
    s = device.Sorter(n, 4, "radix", "iota", graph=True)
    buf = torch.empty(n, dtype=torch.int32, device="cuda")
    for it in range(4):
        k = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
        buf.copy_(torch.from_numpy(k.view(np.int32)))
        ko, vo = s(buf)
        torch.cuda.synchronize()
        want_k, want_i = oracle.sort_u32(k, with_index=True)
        assert np.array_equal(ko.cpu().numpy().view(np.uint32), want_k), it
        assert np.array_equal(vo.cpu().numpy().view(np.uint32), want_i), it
    assert s._graph is not None and s.launches_per_call >= 3


@pytest.mark.parametrize("n", [1000, 1_000_000, 5_000_003])
def test_bucket_cuda_graph_replay(cuda, oracle, n):
    """Sorter(graph=True) for the bucket sort: replays of the async pipeline,
    status checked after each replay; range errors and the oversized fallback
    still come out of the replay path."""
    import torch

    from paper_1206_3511_b200 import device

    rng = np.random.default_rng(n + 1)
    s = device.Sorter(n, 4, "bucket", "iota", range_bound=U32_MAX, graph=True)
    buf = torch.empty(n, dtype=torch.int32, device="cuda")
    for it in range(4):
        k = (rng.integers(0, 1 << 32, size=n, dtype=np.uint64) if it != 2 else
             rng.integers(0, 1 << 20, size=n, dtype=np.uint64)).astype(np.uint32)  # it 2: oversized span
        buf.copy_(torch.from_numpy(k.view(np.int32)))
        ko, vo = s(buf)
        torch.cuda.synchronize()
        want_k, want_i = oracle.sort_u32(k, with_index=True)
        assert np.array_equal(ko.cpu().numpy().view(np.uint32), want_k), it
        assert np.array_equal(vo.cpu().numpy().view(np.uint32), want_i), it
    assert s._graph is not None
    bounded = device.Sorter(n, 4, "bucket", None, range_bound=1000, graph=True)
    buf.copy_(torch.from_numpy(np.arange(n, dtype=np.int32) + 5))  # keys past 1000
    for _ in range(3):  # eager, capture, replay: the range error every time
        with pytest.raises(isort.InvalidArgument, match="exceeds range bound 1000"):
            bounded(buf)


def test_key_range_protocol_single_rank_gpu(cuda, oracle):
    """World size 1 through the same protocol object (no exchange), GPU kernels."""
    import torch

    from paper_1206_3511_b200.partition import CudaOps, KeyRangeSorter

    class OneRank:
        def get_world_size(self):
            return 1

        def get_rank(self):
            return 0

    k = oracle.mixture_u32(2_000_000, 7)
    want_k, want_i = oracle.sort_u32(k, with_index=True)
    tk = torch.from_numpy(k.view(np.int32)).cuda()
    tv = torch.arange(k.size, dtype=torch.int32, device="cuda")
    for alg in ("radix", "bucket"):
        sk, sv, _ = KeyRangeSorter(OneRank(), CudaOps(torch.device("cuda:0"))).sort(tk, tv, algorithm=alg)
        assert np.array_equal(sk.cpu().numpy().view(np.uint32), want_k)
        assert np.array_equal(sv.cpu().numpy().view(np.uint32), want_i)


# ------------------------------------------------------- reverse-sorted early-out (K1 ascents == 0)
@pytest.mark.parametrize("n", [2, 3, 4095, 4096, 4097, 3 * 4096 + 1, 100_003, 1_000_000, 5_000_011])
def test_reverse_sorted_early_out_is_stable(cuda, oracle, n):
    """Non-increasing input takes the run-wise reversal instead of digit passes:
    keys with runs of equal values (short runs, runs across 4096-key tiles, one
    run of everything) must come out with their positions in input order."""
    rng = np.random.default_rng(n)
    cases = {
        "distinct": np.sort(rng.choice(1 << 32, size=n, replace=False).astype(np.uint32))[::-1],
        "short_runs": np.sort(rng.integers(0, max(2, n // 3), size=n, dtype=np.uint64).astype(np.uint32))[::-1],
        "long_runs": np.sort(rng.integers(0, 5, size=n, dtype=np.uint64).astype(np.uint32))[::-1],
        "constant": np.full(n, 7, dtype=np.uint32),
        # runs around the short/long fix-up boundary (kRevShortRun = 64)
        "run_lengths": np.repeat(np.arange(20_000, 0, -1, dtype=np.uint32),
                                 np.resize([1, 2, 63, 64, 65, 66, 127, 128, 129, 3, 5000], 20_000))[:n],
    }
    for name, k in cases.items():
        k = np.ascontiguousarray(k)
        want_k, want_i = oracle.sort_u32(k, with_index=True)
        for alg in ("radix", "bucket"):
            got_k, got_i = dev_sort(k, alg, "iota", range_bound=U32_MAX)
            assert np.array_equal(got_k, want_k), (name, alg, n)
            assert np.array_equal(got_i, want_i), (name, alg, n)
            got_k, _ = dev_sort(k, alg, None, range_bound=U32_MAX)
            assert np.array_equal(got_k, want_k), (name, alg, n, "keys only")
        # a loaded payload follows its key
        pay = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
        import torch

        from paper_1206_3511_b200 import device

        s = device.Sorter(n, 4, "radix", "load")
        ko, vo = s(torch.from_numpy(k.view(np.int32)).cuda(), torch.from_numpy(pay.view(np.int32)).cuda())
        assert np.array_equal(vo.cpu().numpy().view(np.uint32), pay[want_i]), (name, n, "load")


def test_one_ascent_takes_the_digit_passes(cuda, oracle):
    k = np.sort(np.random.default_rng(3).integers(0, 1 << 32, size=50_000, dtype=np.uint64).astype(np.uint32))[::-1]
    k = np.ascontiguousarray(k)
    k[25_000], k[25_001] = k[25_001], k[25_000]  # one ascent: not non-increasing any more
    want_k, want_i = oracle.sort_u32(k, with_index=True)
    got_k, got_i = dev_sort(k, "radix", "iota")
    assert np.array_equal(got_k, want_k) and np.array_equal(got_i, want_i)


# ------------------------------------------------------- Records drop-in: staged multi-chunk transfers
@pytest.mark.parametrize("n,bits", [(3_000_001, 32), (2_500_003, 40), (1_048_576, 20)])
def test_records_staged_transfer_many_chunks(cuda, oracle, n, bits):
    """radix_sort_lsd / bucket_sort on Records big enough to span many 16 MB
    staging chunks and every transfer worker (u32 and u64 key paths)."""
    rng = np.random.default_rng(n)
    seq = recs(rng.integers(0, 1 << bits, size=n, dtype=np.uint64))
    want = oracle.radix_sort_lsd(seq, 256)
    assert np.array_equal(isort.radix_sort_lsd(seq, 256), want)
    assert np.array_equal(isort.bucket_sort(seq, (1 << bits) - 1), want)


# ------------------------------------------------------- host C-ABI entry points (the bench's e2e path)
@pytest.mark.parametrize("n", [0, 1, 4097, 1_000_003])
def test_host_entry_points_bit_exact(cuda, oracle, n):
    """isort_radix_sort_host_u32 / isort_bucket_sort_host_u32: host keys in,
    host keys out (bench.py's e2e call), bit-exact against the oracle, for
    pageable and pinned host buffers."""
    import ctypes

    import torch

    from paper_1206_3511_b200 import _lib

    lib = _lib.load()
    keys = oracle.uniform_u32(n, 7) if n else np.empty(0, dtype=np.uint32)
    want = oracle.sort_u32(keys) if n else keys
    for pinned in (False, True):
        if pinned:
            hin = torch.from_numpy(keys.view(np.int32).copy()).pin_memory()
            hout = torch.empty(max(n, 1), dtype=torch.int32).pin_memory()
            pin_, pout = hin.data_ptr() if n else None, hout.data_ptr()
            got = lambda: hout.numpy()[:n].view(np.uint32)  # noqa: E731
        else:
            src = np.ascontiguousarray(keys)
            dst = np.zeros(max(n, 1), dtype=np.uint32)
            pin_, pout = src.ctypes.data_as(ctypes.c_void_p).value, dst.ctypes.data
            got = lambda: dst[:n]  # noqa: E731
        _lib.check(lib.isort_radix_sort_host_u32(pin_, pout, n, 0))
        assert np.array_equal(got(), want), ("radix", n, pinned)
        _lib.check(lib.isort_bucket_sort_host_u32(pin_, pout, n, U32_MAX, 0))
        assert np.array_equal(got(), want), ("bucket", n, pinned)


def test_host_bucket_entry_reports_range_error(cuda):
    from paper_1206_3511_b200 import _lib

    lib = _lib.load()
    keys = np.array([5, 1, 900, 3, 901], dtype=np.uint32)
    out = np.zeros_like(keys)
    rc = lib.isort_bucket_sort_host_u32(keys.ctypes.data, out.ctypes.data, keys.size, 899, 0)
    assert rc != 0
    assert b"900" in lib.isort_last_error()


@pytest.mark.parametrize("n", [0, 1, 2, 4, 5, 4096, 4097, 1_000_003])
def test_is_sorted_u32(cuda, n):
    """isort_is_sorted_u32 (verify::is_sorted, verify.cpp:67-74): true on sorted
    and constant input, false with one inversion anywhere (first pair, last pair,
    a vector boundary), true for n <= 1."""
    import torch

    from paper_1206_3511_b200 import device

    rng = np.random.default_rng(n)
    k = np.sort(rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32))
    t = torch.from_numpy(k.view(np.int32)).cuda()
    assert device.is_sorted_u32(t) is True
    assert device.is_sorted_u32(torch.zeros(n, dtype=torch.int32, device="cuda")) is True
    if n < 2:
        return
    for pos in sorted({0, n - 2, min(3, n - 2), min(n // 2, n - 2)}):
        bad = k.copy()
        if bad[pos] == 0:
            bad[pos] = 1
        bad[pos + 1] = bad[pos] - np.uint32(1)  # one inversion at (pos, pos + 1)
        assert bad[pos] > bad[pos + 1]
        tb = torch.from_numpy(bad.view(np.int32)).cuda()
        assert device.is_sorted_u32(tb) is False, (n, pos)


# ------------------------------------------------------- small key range: the counting pass (K6)
@pytest.mark.parametrize("n", [1, 2, 5, 4097, 100_003, 4_194_304, 5_000_011])
@pytest.mark.parametrize("top", [2, 1023, 4095, 4096])
def test_counting_pass_small_range(cuda, oracle, n, top):
    """Keys-only sorts of at least 2^22 keys with every key < 2^12 take one
    counting pass (histogram + fill) -- radix always, bucket when M < 2^12 <= n
    (one value per bucket); smaller ones the digit passes.
    max = 4096 must take the digit passes.  Bit-exact against the oracle; with a
    payload the same inputs take the stable scatter."""
    rng = np.random.default_rng(n * 7 + top)
    k = rng.integers(0, top + 1, size=n, dtype=np.uint64).astype(np.uint32)
    if n >= 2:
        k[rng.integers(0, n)] = top  # the maximum is present
    want_k, want_i = oracle.sort_u32(k, with_index=True)
    got_k, _ = dev_sort(k, "radix", None)
    assert np.array_equal(got_k, want_k)
    for bound in (top, max(top, 4095), U32_MAX):
        got_k, _ = dev_sort(k, "bucket", None, range_bound=bound)
        assert np.array_equal(got_k, want_k), bound
    got_k, got_i = dev_sort(k, "radix", "iota")
    assert np.array_equal(got_k, want_k) and np.array_equal(got_i, want_i)


def test_counting_pass_graph_replay_and_reuse(cuda, oracle):
    """The counting path inside a captured graph, alternating with a wide-range
    input on the same Sorter (the plan is decided on the device every call)."""
    import torch

    from paper_1206_3511_b200 import device

    n = 4_200_001
    small = oracle.uniform_u32(n, 3) & np.uint32(1023)
    wide = oracle.uniform_u32(n, 4)
    s = device.Sorter(n, 4, "radix", None, graph=True)
    ts = torch.from_numpy(small.view(np.int32)).cuda()
    tw = torch.from_numpy(wide.view(np.int32)).cuda()
    for _ in range(3):
        for t, k in ((ts, small), (tw, wide)):
            got, _ = s(t)
            torch.cuda.synchronize()
            assert np.array_equal(got.cpu().numpy().view(np.uint32), np.sort(k))


@pytest.mark.parametrize("algorithm", ["radix", "bucket"])
def test_graph_replay_on_caller_stream(cuda, oracle, algorithm):
    """Sorter(graph=True) called with an explicit stream: the replay, the bucket
    status read and its finish all run on that stream."""
    import torch

    from paper_1206_3511_b200 import device

    n = 300_007
    k = oracle.uniform_u32(n, 11)
    t = torch.from_numpy(k.view(np.int32)).cuda()
    s = device.Sorter(n, 4, algorithm, "iota", graph=True)
    want_k, want_i = oracle.sort_u32(k, with_index=True)
    st = torch.cuda.Stream()
    for _ in range(4):
        st.wait_stream(torch.cuda.current_stream())
        ko, vo = s(t, stream=st)
        st.synchronize()
        assert np.array_equal(ko.cpu().numpy().view(np.uint32), want_k)
        assert np.array_equal(vo.cpu().numpy().view(np.uint32), want_i)


def _bucket_passes_executed(keys_np, vals="iota"):
    """Sort on the device with the per-phase profile on; returns (keys, positions,
    number of executed digit passes reported by the plan)."""
    import ctypes

    import torch

    from paper_1206_3511_b200 import _lib, device

    lib = _lib.load()
    t = torch.from_numpy(keys_np.view(np.int32)).cuda()
    s = device.Sorter(keys_np.size, 4, "bucket", vals, range_bound=U32_MAX)
    torch.cuda.synchronize()
    lib.isort_profile_begin()
    k, v = s(t)
    torch.cuda.synchronize()
    ms = (ctypes.c_float * 256)()
    names = ctypes.create_string_buffer(256 * 16)
    cnt, na = ctypes.c_int(0), ctypes.c_int(0)
    _lib.check(lib.isort_profile_end(ms, names, 16, 256, ctypes.byref(cnt), ctypes.byref(na)))
    return k.cpu().numpy().view(np.uint32), (v.cpu().numpy().view(np.uint32) if v is not None else None), na.value


@pytest.mark.parametrize("n", [5_000_011, 20_000_003])
def test_bucket_adaptive_fine_pass_on_skew(cuda, oracle, n):
    """Skewed keys (a dense normal cluster) make K2 run the optional fine bucket
    pass (super-buckets 256x smaller) instead of sending the cluster to the radix
    fallback; uniform keys keep the coarse plan.  Both bit-exact."""
    rng = np.random.default_rng(n)
    skew = np.clip(np.rint(2.0**31 + 2.0**22 * rng.standard_normal(n)), 0, U32_MAX).astype(np.uint32)
    uni = oracle.uniform_u32(n, 5)
    for keys, want_passes in ((skew, 3), (uni, 2)):
        want_k, want_i = oracle.sort_u32(keys, with_index=True)
        got_k, got_i, passes = _bucket_passes_executed(keys)
        assert np.array_equal(got_k, want_k) and np.array_equal(got_i, want_i)
        assert passes == want_passes, (n, passes)
