"""Per-CUDA-source-line instruction and stall totals of an .ncu-rep (needs -lineinfo
and --import-source on):  python tools/ncu_lines.py REP [--top 40] [--kernel REGEX]
(--kernel keeps one kernel of a multi-kernel report, so its lines are not mixed with another's)"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
kern = ["-k", "regex:" + sys.argv[sys.argv.index("--kernel") + 1]] if "--kernel" in sys.argv else []
txt = subprocess.run(["ncu", "-i", rep, *kern, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg, hdr, path = {}, None, ""


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return 0.0


for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":  # a source line row (SASS rows carry an address)
        key = (path, int(r[0]), r[1].strip()[:80])
        a = agg.setdefault(key, [0.0, 0.0])
        a[0] += num(r[hdr.index("Instructions Executed")])
        a[1] += num(r[hdr.index("Warp Stall Sampling (All Samples)")])
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {ti / 1e6:.1f}M, stall samples {ts:.0f}")
for (p, ln, src), (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * i / ti:5.1f}% inst {100 * s / ts:5.1f}% stall  {p}:{ln:<5} {src}")
