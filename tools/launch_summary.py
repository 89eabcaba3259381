"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel.

    python tools/launch_summary.py gpurun_out/launches_bench.csv "command line" > profiles/...txt
"""
import collections
import csv
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
agg = collections.OrderedDict()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].replace("void ", "").replace("unsigned int", "u32").split("(")[0][:60]
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(
        r.get("Metric Unit", "us"), 1e-3)
    t = float(r["Metric Value"].replace(",", "")) * scale
    c, s = agg.get(name, (0, 0.0))
    agg[name] = (c + 1, s + t)
tot = sum(s for _, s in agg.values())
print(f"# ncu launch list of `{sys.argv[2] if len(sys.argv) > 2 else '?'}` (B200, --clock-control none)")
print("# per-launch times are cold-cache and serialised: compare SHARES, not absolutes")
print(f"{'kernel':60} {'launches':>8} {'total_ms':>9} {'share':>6} {'avg_ms':>8}")
for name, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:60} {c:8d} {s:9.3f} {s / tot * 100:5.1f}% {s / c:8.4f}")
