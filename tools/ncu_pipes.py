"""L1TEX data-pipe wavefronts (shared: atom/ld/st, global), pipe utilisation and
warp-stall reasons of each kernel in an .ncu-rep, normalised per 32 keys when
--keys is given.

    python tools/ncu_pipes.py REP [--keys N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
keys = float(sys.argv[sys.argv.index("--keys") + 1]) if "--keys" in sys.argv else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


for row in rows[2:]:
    d = dict(zip(hdr, row))
    print(d.get("Kernel Name", "?")[:110])
    t_us = num(d.get("gpu__time_duration.sum"))
    print(f"  duration {t_us:.2f} us   DRAM {num(d['dram__bytes_read.sum']) + num(d['dram__bytes_write.sum']):.1f} MB")
    per = (keys / 32.0) if keys else None
    for k in ["l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
              "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_st.sum", "smsp__inst_executed.sum"]:
        v = num(d.get(k))
        extra = f"   {v / per:7.2f} per 32 keys" if per else ""
        print(f"  {k:70} {v:14.0f}{extra}")
    sms = 148
    for k in ["SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_shared.avg",
              "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg"]:
        v = num(d.get(k))
        extra = f"   {v * sms / per:7.2f} per 32 keys" if per else ""
        print(f"  {k:70} {v:14.0f}{extra}")
    for k in ["l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread"]:
        print(f"  {k:70} {num(d.get(k)):10.2f}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(v) for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(v for v in st.values() if v == v) or 1
    print("  stalls: " + ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])
                                   if v / tot > 0.01))
