"""Pin the oracle (oracle/isort_oracle.c) before trusting it.

1. Known-answer tests of the reference's own suites, restated
   (proj/tests/test_rng.cpp, test_sort.cpp, test_verify.cpp).
2. Golden vectors produced by the unmodified reference compiled here
   (tests/golden/make_golden.py -> reference_vectors.npz / .json).
3. Where oracle/_ref exists (the build container), a randomized cross-check
   against the reference library itself.
CPU only.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from oracle.binding import RECORD_DTYPE, OracleError, Reference

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
U32_MAX = (1 << 32) - 1


def seq_of(keys):
    a = np.empty(len(keys), dtype=RECORD_DTYPE)
    a["key"] = np.asarray(keys, dtype=np.uint64)
    a["tag"] = np.arange(len(keys), dtype=np.uint64)
    return a


def keys(a):
    return [int(x) for x in a["key"]]


def tags(a):
    return [int(x) for x in a["tag"]]


# ------------------------------------------------------- known answers
def test_splitmix_reference_stream(oracle):  # test_rng.cpp:12-18
    assert oracle.splitmix_stream(0, 3) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_counter_form_matches_generator(oracle):
    g = oracle.generate(1, 1000, U32_MAX, 42)
    assert keys(g)[:3] == [803958421, 2993090819, 319790930]
    assert np.array_equal(oracle.uniform_u32(1000, 42), g["key"].astype(np.uint32))
    g10 = oracle.generate(1, 1000, 1023, 42)
    assert keys(g10)[:3] == [661, 259, 850]
    assert np.array_equal(oracle.uniform_u32(1000, 42, bits=10), g10["key"].astype(np.uint32))


def test_insertion_sort_known_answers(oracle):  # test_sort.cpp:19-34
    assert oracle.insertion_sort(seq_of([])).size == 0
    assert keys(oracle.insertion_sort(seq_of([3, 1, 2]))) == [1, 2, 3]
    out = oracle.insertion_sort(seq_of([2, 1, 2]))
    assert keys(out) == [1, 2, 2] and tags(out) == [1, 0, 2]


def test_counting_pass_known_answers(oracle):  # test_sort.cpp:36-46
    s = seq_of([170, 45, 75])
    assert keys(oracle.counting_sort_by_digit(s, 10, 3, 0)) == [170, 45, 75]
    assert keys(oracle.counting_sort_by_digit(s, 10, 3, 1)) == [45, 170, 75]
    with pytest.raises(OracleError, match="out of range"):
        oracle.counting_sort_by_digit(s, 10, 3, 3)


def test_extract_digit_known_answers(oracle):  # test_sort.cpp:68-75
    assert [oracle.extract_digit(170, i, 10) for i in range(4)] == [0, 7, 1, 0]
    assert oracle.extract_digit(0, 0, 2) == 0
    with pytest.raises(OracleError):
        oracle.extract_digit(1, 0, 1)


def test_build_radix_plan_known_answers(oracle):  # test_sort.cpp:95-105
    assert oracle.build_radix_plan(seq_of([0]), 10) == 1
    assert oracle.build_radix_plan(seq_of([]), 10) == 1
    assert oracle.build_radix_plan(seq_of([0, 0, 0]), 7) == 1
    assert oracle.build_radix_plan(seq_of([999_999]), 10) == 6
    assert oracle.build_radix_plan(seq_of([100_000_000]), 10) == 9
    assert oracle.build_radix_plan(seq_of([1_000_000]), 10) == 7
    assert oracle.build_radix_plan(seq_of([255]), 256) == 1
    assert oracle.build_radix_plan(seq_of([256]), 256) == 2
    with pytest.raises(OracleError):
        oracle.build_radix_plan(seq_of([1]), 1)


def test_radix_known_answer(oracle):  # test_sort.cpp:124-134
    s = seq_of([170, 45, 75, 90, 802, 24, 2, 66])
    out = oracle.radix_sort_lsd(s, 10)
    assert keys(out) == [2, 24, 45, 66, 75, 90, 170, 802]
    assert (out == oracle.oracle_sort(s)).all()
    assert (oracle.radix_sort_lsd(s, 256) == out).all()
    with pytest.raises(OracleError):
        oracle.radix_sort_lsd(s, 1)


def test_bucket_index_known_answers(oracle):  # test_sort.cpp:151-174
    assert oracle.bucket_index(0, 10, 999) == 0
    assert oracle.bucket_index(999, 10, 999) == 9
    assert oracle.bucket_index(500, 10, 999) == 5
    with pytest.raises(OracleError, match="exceeds range bound"):
        oracle.bucket_index(1000, 10, 999)
    with pytest.raises(OracleError):
        oracle.bucket_index(0, 0, 999)
    assert oracle.bucket_index(1 << 40, 1 << 32, 1 << 40) == (1 << 32) - 1
    assert oracle.bucket_index(0, 1 << 32, 1 << 40) == 0


def test_bucket_sort_known_answers(oracle):  # test_sort.cpp:185-192
    assert oracle.bucket_sort(seq_of([]), 100).size == 0
    s = seq_of([1, 2, 2, 3, 10])
    assert (oracle.bucket_sort(s, 10) == s).all()
    with pytest.raises(OracleError):
        oracle.bucket_sort(seq_of([11]), 10)


def test_oracle_exhaustive_small(oracle):  # test_verify.cpp:29-45
    for length in range(7):
        for code in range(3 ** length):
            ks, rest = [], code
            for _ in range(length):
                ks.append(rest % 3)
                rest //= 3
            s = seq_of(ks)
            assert (oracle.oracle_sort(s) == oracle.insertion_sort(s)).all()


def test_keys_only_oracle_is_stable_lsd(oracle):
    rng = np.random.default_rng(1)
    for bits in (32, 10, 1):
        k = rng.integers(0, 1 << bits, size=100_003, dtype=np.uint64).astype(np.uint32)
        ko, idx = oracle.sort_u32(k, with_index=True)
        ref = np.argsort(k, kind="stable")
        assert np.array_equal(idx, ref.astype(np.uint32))
        assert np.array_equal(ko, k[ref])


# ------------------------------------------------------- golden vectors
@pytest.fixture(scope="module")
def golden():
    z = np.load(os.path.join(GOLDEN, "reference_vectors.npz"))
    with open(os.path.join(GOLDEN, "reference_vectors.json")) as f:
        meta = json.load(f)
    return z, meta


def test_oracle_generator_matches_reference_inputs(oracle, golden):
    z, meta = golden
    for i, sp in enumerate(meta):
        g = oracle.generate(sp["case_id"], sp["n"], sp["range_bound"], sp["seed"])
        assert np.array_equal(g["key"], z[f"in_{i}"]), sp


def test_oracle_sorts_match_reference_outputs(oracle, golden):
    z, meta = golden
    for i, sp in enumerate(meta):
        s = seq_of(z[f"in_{i}"])
        assert np.array_equal(oracle.radix_sort_lsd(s, 10)["tag"], z[f"radix10_{i}"]), sp
        assert np.array_equal(oracle.radix_sort_lsd(s, 256)["tag"], z[f"radix256_{i}"]), sp
        assert np.array_equal(oracle.bucket_sort(s, sp["bound"])["tag"], z[f"bucket_{i}"]), sp
        assert oracle.build_radix_plan(s, 10) == sp["digits10"]
        assert oracle.build_radix_plan(s, 256) == sp["digits256"]
        if sp["n"]:
            d = sp["digits10"]
            assert np.array_equal(oracle.counting_sort_by_digit(s, 10, d, d - 1)["tag"], z[f"count_top_{i}"]), sp


def test_oracle_bucket_index_matches_reference(oracle, golden):
    z, _ = golden
    for key, count, bound, want in z["bucket_index"].tolist():
        assert oracle.bucket_index(int(key), int(count), int(bound)) == int(want)


# ------------------------------------------------------- live reference (build container only)
@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built here")
def test_oracle_against_live_reference(oracle):
    ref = Reference()
    rng = np.random.default_rng(99)
    for _ in range(60):
        case_id = int(rng.integers(1, 7))
        n = int(rng.integers(0, 600))
        seed = int(rng.integers(1 << 62))
        s = ref.generate(case_id, n, None, seed)
        assert (oracle.generate(case_id, n, None, seed) == s).all()
        bound = oracle.default_range_bound(case_id)
        assert (oracle.bucket_sort(s, bound) == ref.bucket_sort(s, bound)).all()
        base = int(rng.choice([2, 3, 10, 255, 256, 1000]))
        assert (oracle.radix_sort_lsd(s, base) == ref.radix_sort_lsd(s, base)).all()
