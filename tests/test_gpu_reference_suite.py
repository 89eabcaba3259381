"""The reference's sorting suite (proj/tests/test_sort.cpp), restated in Python
against the GPU-backed drop-in API (paper_1206_3511_b200.intsort).  Each test
cites the reference test it mirrors.  Also runs the reference's own C++ suites
linked against our C++ drop-in (oracle/_ref/dropin_tests) when it was built."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

import paper_1206_3511_b200 as isort
from paper_1206_3511_b200 import keys_of, seq_of, tags_of
from paper_1206_3511_b200.harness import AlgorithmId, make_sort_fn, parse_algorithm, time_sort

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def is_sorted(s):
    k = s["key"]
    return bool(np.all(k[:-1] <= k[1:])) if k.size > 1 else True


def is_permutation(a, b):
    return a.size == b.size and np.array_equal(np.sort(a, order=["key", "tag"]), np.sort(b, order=["key", "tag"]))


def is_stable(a, b):
    """verify.cpp:109-115: per key, tags in the same relative order."""
    assert is_permutation(a, b)
    ia = np.argsort(a["key"], kind="stable")
    return np.array_equal(a["tag"][ia], b["tag"])


def test_insertion_sort(cuda):  # test_sort.cpp:19-34
    assert isort.insertion_sort(seq_of([])).size == 0
    assert keys_of(isort.insertion_sort(seq_of([3, 1, 2]))) == [1, 2, 3]
    out = isort.insertion_sort(seq_of([2, 1, 2]))
    assert keys_of(out) == [1, 2, 2] and tags_of(out) == [1, 0, 2]
    src = seq_of([5, 4, 3])
    copy = src.copy()
    isort.insertion_sort(src)
    assert (src == copy).all()


def test_counting_sort_by_digit(cuda):  # test_sort.cpp:36-66
    plan = isort.RadixPlan(10, 3)
    s = seq_of([170, 45, 75])
    assert keys_of(isort.counting_sort_by_digit(s, plan, 0)) == [170, 45, 75]
    assert keys_of(isort.counting_sort_by_digit(s, plan, 1)) == [45, 170, 75]
    with pytest.raises(isort.InvalidArgument):
        isort.counting_sort_by_digit(s, plan, 3)
    rng = np.random.default_rng(2024)
    for _ in range(50):
        n = int(rng.integers(0, 200))
        s = seq_of(rng.integers(0, 100_000, size=n))
        p = isort.build_radix_plan(s, 10)
        d = int(rng.integers(0, p.digits))
        out = isort.counting_sort_by_digit(s, p, d)
        assert sorted(keys_of(out)) == sorted(keys_of(s))
        digits = [(k // 10**d) % 10 for k in keys_of(out)]
        assert digits == sorted(digits)


def test_build_radix_plan(cuda):  # test_sort.cpp:95-122
    assert isort.build_radix_plan(seq_of([0]), 10).digits == 1
    assert isort.build_radix_plan(seq_of([]), 10).digits == 1
    assert isort.build_radix_plan(seq_of([999_999]), 10).digits == 6
    assert isort.build_radix_plan(seq_of([100_000_000]), 10).digits == 9
    assert isort.build_radix_plan(seq_of([255]), 256).digits == 1
    assert isort.build_radix_plan(seq_of([256]), 256).digits == 2
    rng = np.random.default_rng(11)
    for _ in range(100):
        key = int(rng.integers(0, 1 << 40))
        base = int(rng.integers(2, 102))
        d = isort.build_radix_plan(seq_of([key, key // 2]), base).digits
        low = base ** (d - 1)
        if key > 0:
            assert key >= low
        assert key < low * base


def test_radix_sort_lsd_any_base(cuda, oracle):  # test_sort.cpp:124-149
    assert isort.radix_sort_lsd(seq_of([]), 10).size == 0
    s = seq_of([170, 45, 75, 90, 802, 24, 2, 66])
    out = isort.radix_sort_lsd(s, 10)
    assert keys_of(out) == [2, 24, 45, 66, 75, 90, 170, 802]
    assert (out == oracle.oracle_sort(s)).all()
    assert (isort.radix_sort_lsd(s, 256) == out).all()
    with pytest.raises(isort.InvalidArgument):
        isort.radix_sort_lsd(s, 1)
    rng = np.random.default_rng(99)
    for _ in range(20):
        case_id = int(rng.integers(1, 7))
        sp = oracle.generate(case_id, int(rng.integers(0, 500)), None, int(rng.integers(1 << 62)))
        b10 = isort.radix_sort_lsd(sp, 10)
        for base in (2, 256, 1000):
            assert (isort.radix_sort_lsd(sp, base) == b10).all()


def test_bucket_sort_matches_oracle(cuda, oracle):  # test_sort.cpp:185-204
    assert isort.bucket_sort(seq_of([]), 100).size == 0
    s = seq_of([1, 2, 2, 3, 10])
    assert (isort.bucket_sort(s, 10) == s).all()
    with pytest.raises(isort.InvalidArgument):
        isort.bucket_sort(seq_of([11]), 10)
    rng = np.random.default_rng(123)
    for _ in range(300):
        case_id = int(rng.integers(1, 7))
        sp = oracle.generate(case_id, int(rng.integers(0, 300)), None, int(rng.integers(1 << 62)))
        bound = oracle.default_range_bound(case_id)
        assert (isort.bucket_sort(sp, bound) == oracle.oracle_sort(sp)).all()


def test_sorting_sorted_is_identity(cuda, oracle):  # test_sort.cpp:206-218
    rng = np.random.default_rng(321)
    for _ in range(30):
        case_id = int(rng.integers(1, 7))
        once = isort.radix_sort_lsd(oracle.generate(case_id, int(rng.integers(0, 400)), None,
                                                    int(rng.integers(1 << 62))), 10)
        assert (isort.radix_sort_lsd(once, 10) == once).all()
        assert (isort.bucket_sort(once, oracle.default_range_bound(case_id)) == once).all()
        assert (isort.insertion_sort(once) == once).all()


def test_stable_permutations(cuda, oracle):  # test_sort.cpp:220-236
    rng = np.random.default_rng(777)
    for _ in range(150):
        case_id = int(rng.integers(1, 7))
        sp = oracle.generate(case_id, int(rng.integers(0, 250)), None, int(rng.integers(1 << 62)))
        bound = oracle.default_range_bound(case_id)
        for out in (isort.insertion_sort(sp), isort.bucket_sort(sp, bound), isort.radix_sort_lsd(sp, 10)):
            assert is_sorted(out) and is_permutation(sp, out) and is_stable(sp, out)


def test_records_with_40_bit_keys(cuda, oracle):  # record.hpp:15, generator up to 2^40
    rng = np.random.default_rng(40)
    for n in (1, 1000, 50_001):
        sp = oracle.generate(1, n, 1 << 40, int(rng.integers(1 << 62)))
        want = oracle.oracle_sort(sp)
        assert (isort.radix_sort_lsd(sp, 10) == want).all()
        assert (isort.bucket_sort(sp, 1 << 40) == want).all()


def test_harness_registry_and_timer(cuda, oracle):  # bench.hpp:15-66, bench.cpp:42-99
    assert parse_algorithm("radix") is AlgorithmId.radix and parse_algorithm("nope") is None
    sp = oracle.generate(1, 10_000, None, 1)
    for alg in AlgorithmId:
        fn = make_sort_fn(alg, oracle.default_range_bound(1), 10)
        assert (fn(sp) == oracle.oracle_sort(sp)).all()
        st = time_sort(fn, sp, 3)
        assert st.median_s > 0
    with pytest.raises(ValueError):
        time_sort(make_sort_fn(AlgorithmId.radix, 0, 10), sp, 2)


DROPIN_TESTS = os.path.join(ROOT, "oracle", "_ref", "dropin_tests")


@pytest.mark.skipif(not os.path.exists(DROPIN_TESTS), reason="drop-in C++ suite not built (needs /root/reference)")
def test_reference_cpp_suites_against_dropin(cuda):
    """The reference's own test_sort/test_verify/test_rng/test_generator, compiled
    unchanged with our doctest shim and linked against the GPU drop-in sort.cpp
    replacement (paper_1206_3511_b200/dropin/sort_b200.cpp)."""
    r = subprocess.run([DROPIN_TESTS], capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, LD_LIBRARY_PATH=os.path.join(ROOT, "paper_1206_3511_b200")))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed: 0" in r.stdout
