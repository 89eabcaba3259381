"""GPU rows for the reference's benchmark matrix and report.

Mirrors proj/core/src/bench.cpp (run_matrix, bench.cpp:105-154) and
proj/core/src/report.cpp (emit_csv, compute_scaling_fits, report.cpp:17,
318-396) for the device engine:

* ``run_matrix(config)`` -- every (case, n, algorithm) cell: the reference's own
  input (``inputs.generate_case``, exact), keys resident on the GPU, one checked
  warm-up, ``repeats`` runs timed with CUDA events, median and relative spread
  (bench.cpp:67-99).  ``config.range_bound`` is honoured (bench.cpp:132 ignores
  it and always uses the case default).
* ``emit_csv`` -- the reference's columns ``algorithm,case,n,median_time_s,
  relative_spread,peak_bytes`` (peak_bytes = device bytes held by the sort), then
  ``device,n_gpus,gkeys_per_s,gb_per_s,roofline_frac``: throughput, algorithmic
  HBM bytes / time (keys-only: 4n + 8n per executed pass, bucket + 8n for the
  segment sort), and that over the measured copy peak.
* ``compute_scaling_fits`` -- log-log least squares of median time against n per
  (algorithm, case), as report.cpp does, over the GPU rows.

    python -m paper_1206_3511_b200.report --cases 1,4,6 --sizes 1e6,1e7 --csv out.csv
"""
from __future__ import annotations

import argparse
import io
import json
import math
import os
import sys
from dataclasses import dataclass, field

import numpy as np

CSV_HEADER = ("algorithm,case,n,median_time_s,relative_spread,peak_bytes,"
              "device,n_gpus,gkeys_per_s,gb_per_s,roofline_frac")
DISPLAY_RANK = {"radix": 0, "bucket": 1, "insertion": 2}  # report.cpp:22-32


@dataclass
class BenchConfig:  # bench.hpp BenchConfig
    cases: list[int] = field(default_factory=lambda: [1, 2, 3, 4, 5, 6])
    sizes: list[int] = field(default_factory=lambda: [10**5, 10**6, 10**7])
    algorithms: list[str] = field(default_factory=lambda: ["radix", "bucket"])
    repeats: int = 5
    seed: int = 42
    radix_base: int = 256
    range_bound: int | None = None  # honoured (None: the case's default bound)


@dataclass
class BenchResult:
    algorithm: str
    case_id: int
    n: int
    median_time_s: float
    relative_spread: float
    peak_bytes: int
    device: str = "b200"
    n_gpus: int = 1
    gkeys_per_s: float = 0.0
    gb_per_s: float = 0.0
    roofline_frac: float = 0.0


@dataclass
class CellError:
    algorithm: str
    case_id: int
    n: int
    message: str


def _peak_gbs() -> float:
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0  # B200_PROFILING.md fallback


def _algorithmic_bytes(alg: str, n: int, key_bytes: int, passes: int) -> int:
    b = key_bytes * n + 2 * key_bytes * n * passes
    return b + 2 * key_bytes * n if alg == "bucket" else b


def time_cell(alg: str, keys_np: np.ndarray, range_bound: int, repeats: int):
    """(median s, relative spread, device bytes, executed passes) of one cell."""
    import torch

    from . import device

    if repeats < 3:
        raise ValueError("run_matrix: repeats must be >= 3")
    kb = 4 if (keys_np.size == 0 or int(keys_np.max()) < (1 << 32)) else 8
    host = keys_np.astype(np.uint32 if kb == 4 else np.uint64)
    keys = torch.from_numpy(host.view(np.int32 if kb == 4 else np.int64)).cuda()
    algo = "bucket" if alg == "bucket" else "radix"  # insertion: the unique stable sort, via radix
    s = device.Sorter(keys.numel(), kb, algo, None, range_bound=range_bound)
    view = np.uint32 if kb == 4 else np.uint64
    s(keys)  # checked warm-up (bench.cpp:73-76)
    torch.cuda.synchronize()
    w = s.keys_out.cpu().numpy().view(view)
    if w.size > 1 and not bool(np.all(w[1:] >= w[:-1])):
        raise RuntimeError("time_sort: warm-up run produced unsorted output")
    times = []
    for _ in range(repeats):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s(keys)
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b) / 1e3)
    got = s.keys_out.cpu().numpy().view(view)
    if not np.array_equal(got, np.sort(host)):
        raise RuntimeError("time_sort: timed run produced unsorted output, measurement rejected")
    times.sort()
    c = len(times)
    med = times[c // 2] if c % 2 else 0.5 * (times[c // 2 - 1] + times[c // 2])
    spread = (times[-1] - times[0]) / med if med > 0 else 0.0
    st_bytes = s.temp_bytes + 2 * kb * keys.numel()
    # executed passes: the plan skips trivial digits and sorted inputs
    max_key = int(host.max()) if host.size else 0
    digits = max(1, (max_key.bit_length() + 7) // 8)
    sorted_in = bool(np.all(host[1:] >= host[:-1])) if host.size > 1 else True
    passes = 0 if sorted_in else digits
    return med, spread, st_bytes, passes, kb


def run_matrix(config: BenchConfig, errors: list | None = None, generate=None) -> list[BenchResult]:
    """bench.cpp:105-154 for the device engine; `generate(case, n, bound, seed)` -> keys."""
    from . import inputs

    if config.repeats < 3:
        raise ValueError("run_matrix: repeats must be >= 3")
    gen = generate or (lambda c, n, b, s: inputs.generate_case(c, n, b, s))
    peak = _peak_gbs()
    results = []
    for case_id in sorted(config.cases):
        for n in sorted(config.sizes):
            bound = config.range_bound if config.range_bound is not None else inputs.default_range_bound(case_id)
            try:
                keys = gen(case_id, n, bound, config.seed)
            except Exception as e:  # noqa: BLE001 - mirrors CellError collection
                if errors is None:
                    raise RuntimeError(f"[{case_id}, n={n}] generation failed: {e}") from e
                errors.extend(CellError(a, case_id, n, str(e)) for a in config.algorithms)
                continue
            for alg in config.algorithms:
                try:
                    med, spread, peak_bytes, passes, kb = time_cell(alg, keys, bound, config.repeats)
                    gbs = _algorithmic_bytes(alg, n, kb, passes) / med / 1e9 if med > 0 else 0.0
                    results.append(BenchResult(alg, case_id, n, med, spread, peak_bytes,
                                               gkeys_per_s=n / med / 1e9 if med > 0 else 0.0, gb_per_s=gbs,
                                               roofline_frac=gbs / peak))
                except Exception as e:  # noqa: BLE001
                    if errors is None:
                        raise
                    errors.append(CellError(alg, case_id, n, str(e)))
    return results


def emit_csv(results: list[BenchResult], out=None) -> str:
    """Reference columns first (report.cpp:17), rows in (case, n, algorithm) order."""
    buf = io.StringIO()
    buf.write(CSV_HEADER + "\n")
    for r in sorted(results, key=lambda r: (r.case_id, r.n, DISPLAY_RANK.get(r.algorithm, 3))):
        buf.write(f"{r.algorithm},{r.case_id},{r.n},{r.median_time_s:.9g},{r.relative_spread:.6g},{r.peak_bytes},"
                  f"{r.device},{r.n_gpus},{r.gkeys_per_s:.6g},{r.gb_per_s:.6g},{r.roofline_frac:.4f}\n")
    text = buf.getvalue()
    if out is not None:
        out.write(text)
    return text


def parse_csv(text: str) -> list[BenchResult]:
    lines = [l for l in text.splitlines() if l]
    if not lines or lines[0] != CSV_HEADER:
        raise RuntimeError("parse_csv: bad header")
    out = []
    for l in lines[1:]:
        f = l.split(",")
        if len(f) != 11:
            raise RuntimeError(f"parse_csv: malformed row {l!r}")
        out.append(BenchResult(f[0], int(f[1]), int(f[2]), float(f[3]), float(f[4]), int(f[5]), f[6], int(f[7]),
                               float(f[8]), float(f[9]), float(f[10])))
    return out


@dataclass
class ScalingFit:
    algorithm: str = "bucket"
    case_id: int = 0
    slope: float = 0.0
    r_squared: float = 0.0


def fit_loglog_slope(points) -> ScalingFit:  # report.cpp:318-358
    if len(points) < 2:
        raise ValueError("fit_loglog_slope: need at least 2 points")
    if any(n <= 0 or s <= 0 for n, s in points):
        raise ValueError("fit_loglog_slope: points must be positive")
    xs = [math.log(n) for n, _ in points]
    ys = [math.log(s) for _, s in points]
    mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
    sxx = sum((x - mx) ** 2 for x in xs)
    sxy = sum((x - mx) * (y - my) for x, y in zip(xs, ys))
    syy = sum((y - my) ** 2 for y in ys)
    if sxx == 0.0:
        raise ValueError("fit_loglog_slope: need at least 2 distinct n values")
    return ScalingFit(slope=sxy / sxx, r_squared=1.0 if syy == 0.0 else (sxy * sxy) / (sxx * syy))


def compute_scaling_fits(results: list[BenchResult]) -> list[ScalingFit]:  # report.cpp:360-396
    groups: dict = {}
    for r in results:
        groups.setdefault((DISPLAY_RANK.get(r.algorithm, 3), r.case_id), (r.algorithm, []))[1].append(
            (float(r.n), r.median_time_s))
    fits = []
    for (_, case_id), (alg, pts) in sorted(groups.items()):
        if len({n for n, _ in pts}) < 2 or any(n <= 0 or s <= 0 for n, s in pts):
            continue
        f = fit_loglog_slope(sorted(pts))
        f.algorithm, f.case_id = alg, case_id
        fits.append(f)
    return fits


def emit_scaling_report(results: list[BenchResult]) -> str:  # report.cpp:398-416
    fits = compute_scaling_fits(results)
    if not fits:
        return "scaling analysis omitted: need at least two distinct sizes per (algorithm, case) pair\n"
    lines = ["Scaling of median time vs n (log-log least squares; slope 1 = linear)", "",
             "algorithm   case     slope       r^2"]
    lines += [f"{f.algorithm:<11s} {f.case_id:4d} {f.slope:9.3f} {f.r_squared:9.4f}" for f in fits]
    return "\n".join(lines) + "\n"


def main(argv=None) -> int:
    p = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    p.add_argument("--cases", default="1,2,3,4,5,6")
    p.add_argument("--sizes", default="1e5,1e6,1e7")
    p.add_argument("--algorithms", default="radix,bucket")
    p.add_argument("--repeats", type=int, default=5)
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--range-bound", type=int, default=None)
    p.add_argument("--csv", default=None)
    a = p.parse_args(argv)
    cfg = BenchConfig(cases=[int(x) for x in a.cases.split(",")], sizes=[int(float(x)) for x in a.sizes.split(",")],
                      algorithms=a.algorithms.split(","), repeats=a.repeats, seed=a.seed, range_bound=a.range_bound)
    errors: list = []
    res = run_matrix(cfg, errors)
    text = emit_csv(res)
    if a.csv:
        with open(a.csv, "w") as f:
            f.write(text)
    sys.stdout.write(text)
    sys.stdout.write(emit_scaling_report(res))
    for e in errors:
        sys.stderr.write(f"[{e.algorithm} case {e.case_id} n={e.n}] {e.message}\n")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
