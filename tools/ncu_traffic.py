"""Per-launch DRAM traffic of the dominant kernels, from `ncu --set full` captures.

    python tools/ncu_traffic.py OUT.json REP.ncu-rep [REP2.ncu-rep ...]

Writes {kernel_family: {"dram_bytes_per_launch": B, "read": R, "write": W,
"duration_us": T, "source": rep}} for the families bench.py reports
(k_onesweep_t, k_onesweep, k_bucket_segments, k_upfront).  bench.py copies the figure into
its roofline "traffic" field when profiles/ncu_traffic.json exists.
"""
import csv
import io
import json
import os
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1024**2, "GB": 1024**3}
FAMILIES = ("k_onesweep_t", "k_onesweep", "k_bucket_segments", "k_upfront")  # first match wins


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    raw = list(csv.reader(io.StringIO(out)))
    hdr, units = raw[0], raw[1]
    for r in raw[2:]:
        yield dict(zip(hdr, r)), dict(zip(hdr, units))


def main():
    dst, reps = sys.argv[1], sys.argv[2:]
    res = json.load(open(dst)) if os.path.exists(dst) else {}
    for rep in reps:
        for d, u in rows(rep):
            name = d.get("Kernel Name", "")
            fam = next((f for f in FAMILIES if f in name), None)
            if fam is None or fam in res and res[fam].get("source") == os.path.basename(rep):
                continue

            def val(k):
                return float(d[k].replace(",", "")) * SCALE.get(u.get(k, "byte"), 1)

            rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
            res[fam] = {"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr,
                        "duration_us": float(d["gpu__time_duration.sum"].replace(",", ""))
                        * {"nsecond": 1e-3, "msecond": 1e3}.get(u.get("gpu__time_duration.sum"), 1.0),
                        "kernel": name[:120], "source": os.path.basename(rep)}
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
