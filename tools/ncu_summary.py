"""Summarise an .ncu-rep: key throughput metrics + top SASS stall sites + instruction mix.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--top 25]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units = raw[0], raw[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "lts__t_bytes.sum", "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum"]
for row in raw[2:]:
    d = dict(zip(hdr, row))
    u = dict(zip(hdr, units))
    for w in want:
        if w in d:
            print(f"{w:75} {d[w][:100]} {u.get(w, '')}")
    print()

src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
h = src[1]
ix = {k: i for i, k in enumerate(h)}
data = src[2:]
S = "Warp Stall Sampling (All Samples)"


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return 0.0


data = [r for r in data if len(r) == len(h) and r[ix["Source"]] != "Source"]
for r in data:
    r[ix[S]] = num(r[ix[S]])
    r[ix["Instructions Executed"]] = num(r[ix["Instructions Executed"]])
tot = sum(r[ix[S]] for r in data) or 1
print("top stall sites:")
for r in sorted(data, key=lambda r: -r[ix[S]])[:top]:
    print(f"  {r[ix[S]] / tot * 100:5.1f}%  {r[ix['Source']][:70]:70} exec={r[ix['Instructions Executed']]:.0f}")
c = collections.Counter()
for r in data:
    op = r[ix["Source"]].split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    c[o.split(".")[0]] += r[ix["Instructions Executed"]]
t = sum(c.values())
print("instruction mix (warp-level):", f"{t / 1e6:.1f}M total")
print("  " + ", ".join(f"{k} {v / t * 100:.1f}%" for k, v in c.most_common(16)))
