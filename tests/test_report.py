"""SURVEY 8f rows f3/f4 host side: the reference's six input cases (exact, pinned
against the reference itself), the benchmark-matrix CSV and scaling fits for
GPU rows (report.cpp), and a small GPU matrix run."""
from __future__ import annotations

import numpy as np
import pytest

from oracle.binding import Reference
from paper_1206_3511_b200 import inputs, report


@pytest.fixture(scope="module")
def ref():
    if not Reference.available():
        pytest.skip("oracle/_ref (the reference built here) is not present")
    return Reference()


@pytest.mark.parametrize("case_id", [1, 2, 3, 4, 5, 6])
def test_generate_case_is_the_reference_generator(ref, case_id):
    for n in (0, 1, 2, 7, 999, 20_001):
        for seed in (0, 42, 99):
            want = ref.generate(case_id, n, None, seed)["key"]
            assert np.array_equal(inputs.generate_case(case_id, n, None, seed), want), (case_id, n, seed)
    for bound in (1, 1023, 99_991, 1 << 32, 1 << 40):
        try:
            want = ref.generate(case_id, 3000, bound, 5)["key"]
        except Exception:  # noqa: BLE001 - infeasible specs must fail on both sides
            with pytest.raises(ValueError):
                inputs.generate_case(case_id, 3000, bound, 5)
            continue
        assert np.array_equal(inputs.generate_case(case_id, 3000, bound, 5), want), (case_id, bound)


def test_loglog_fit_and_csv_roundtrip():
    rows = [report.BenchResult("radix", 1, n, 1e-9 * n ** 1.1, 0.01, 8 * n, gkeys_per_s=1.0, gb_per_s=2.0,
                               roofline_frac=0.3) for n in (10**5, 10**6, 10**7)]
    rows += [report.BenchResult("bucket", 4, 10**6, 0.001, 0.02, 100)]
    fits = report.compute_scaling_fits(rows)
    assert len(fits) == 1 and fits[0].algorithm == "radix" and fits[0].case_id == 1
    assert abs(fits[0].slope - 1.1) < 1e-9 and abs(fits[0].r_squared - 1.0) < 1e-12
    text = report.emit_csv(rows)
    assert text.splitlines()[0].startswith("algorithm,case,n,median_time_s,relative_spread,peak_bytes,")
    back = report.parse_csv(text)
    assert [(r.algorithm, r.case_id, r.n) for r in back] == [("radix", 1, 10**5), ("radix", 1, 10**6),
                                                              ("radix", 1, 10**7), ("bucket", 4, 10**6)]
    with pytest.raises(ValueError):
        report.fit_loglog_slope([(10.0, 1.0), (10.0, 2.0)])
    assert "omitted" in report.emit_scaling_report(rows[3:])


@pytest.mark.gpu
def test_matrix_gpu_rows(cuda):
    cfg = report.BenchConfig(cases=[1, 3, 6], sizes=[20_000, 200_000], algorithms=["radix", "bucket"], repeats=3)
    errors: list = []
    rows = report.run_matrix(cfg, errors)
    assert not errors and len(rows) == 12
    assert all(r.median_time_s > 0 and r.gkeys_per_s > 0 for r in rows)
    # the override is honoured: a bound below case 1's keys fails the bucket cells (key > M)
    errors = []
    bad = report.run_matrix(report.BenchConfig(cases=[1], sizes=[1000], algorithms=["bucket"], repeats=3,
                                               range_bound=10), errors,
                            generate=lambda c, n, b, s: inputs.generate_case(c, n, None, s))
    assert not bad and errors and "exceeds range bound" in errors[0].message
