#!/usr/bin/env python
"""bench.py -- Gkeys/s sorting 100M uint32 keys (LSD radix & bucket) on B200.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` prints ONE
JSON line on rank 0.  A step = one full sort (one pass of the hot path) of the
configuration's batch of keys.  N=1 workload = BASELINE.json configs[1] (C2:
1e8 u32 keys, uniform over [0, 2^32), seed 42).  N>1 (torchrun, one rank per
GPU): each rank holds 1e8 keys (weak scaling), the job sorts all N*1e8 keys by
key range (sampled-histogram splitters + NCCL all-to-all exchange + local
sort; paper_1206_3511_b200/partition.py).

value  = whole-job keys / device time (CUDA events on the sort's stream, max
         over ranks), inputs resident in HBM.  Headline algorithm: LSD radix;
         the bucket sort is reported in the "bucket" object with the same keys.
e2e    = the same metric through the host C-ABI call (isort_radix_sort_host_u32:
         pinned host keys in, H2D, sort, D2H, synchronous).
roofline = the one-sweep digit pass (dominant kernel): 8n algorithmic bytes per
         launch / its live CUDA-event duration, against MEASURED_PEAKS.json.
cpu_baseline = the reference's own radix_sort_lsd (oracle/_ref, base 256) on
         the host cores, bounded sample.  `--impl reference` runs only that.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gkeys/s sorting 100M uint32 (radix & bucket) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "Gkeys/s"
N_DEFAULT = 100_000_000
FALLBACK_HBM_GBS = 6650.0


def ncu_traffic(family):
    """Per-launch DRAM bytes of a kernel family from a committed `ncu --set full`
    capture (tools/ncu_traffic.py -> profiles/ncu_traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)[family]
        return t["dram_bytes_per_launch"], t["source"]
    except (OSError, KeyError, ValueError):
        return None, None


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="c2", help="c1 c2 c3 c4a c4b c5 (keys per rank)")
    p.add_argument("--n", type=int, default=None, help="keys per rank (default: the config's n)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU-baseline work per thread")
    p.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                   help="replay each sort pipeline as one CUDA graph (auto = on); the phase/roofline loop runs eagerly")
    return p.parse_args()


# ----------------------------------------------------------------- helpers
def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy, burst)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback 6.65 TB/s (B200_PROFILING.md), MEASURED_PEAKS.json absent"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], None, set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for name, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "samples": len(sm),
                "reasons": sorted(reasons)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------- reference arm
def cpu_reference_run(n_sample: int, threads: int, target_s: float, config: str, seed: int = 42):
    """Reference radix_sort_lsd (base 256, 8-bit digits) on `threads` host threads,
    each sorting its own seeded n_sample-key sample of the configuration's
    distribution repeatedly for ~target_s.  Returns (Gkeys/s, info)."""
    import numpy as np

    from oracle.binding import RECORD_DTYPE, Oracle, Reference
    from paper_1206_3511_b200 import inputs

    kind = "reference" if Reference.available() else "port"
    impl = Reference() if kind == "reference" else Oracle()
    samples = []
    for t in range(threads):
        seq = np.empty(n_sample, dtype=RECORD_DTYPE)
        seq["key"] = inputs.config_keys(config, n_sample, seed + 1000 * t).astype(np.uint64) \
            if config not in ("c4a", "c4b") else inputs.config_keys(config, n_sample, seed)
        seq["tag"] = np.arange(n_sample, dtype=np.uint64)
        samples.append(seq)
    # one warm-up sort (not timed) -- mirrors time_sort's warm-up (bench.cpp:73-76)
    impl.radix_sort_lsd(samples[0][: min(n_sample, 100_000)], 256)
    counts = [0] * threads
    stop_at = [0.0]

    def worker(i):
        while True:
            impl.radix_sort_lsd(samples[i], 256)  # ctypes releases the GIL
            counts[i] += 1
            if time.perf_counter() >= stop_at[0]:
                break

    t0 = time.perf_counter()
    stop_at[0] = t0 + target_s
    ths = [threading.Thread(target=worker, args=(i,)) for i in range(threads)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    dt = time.perf_counter() - t0
    keys = sum(counts) * n_sample
    info = {"kind": kind, "cores": threads,
            "sample": (f"{threads} thread(s) x {n_sample:,}-key {config} samples (16-byte Records), "
                       f"reference radix_sort_lsd base 256 (8-bit digits, 4 passes), {sum(counts)} sorts "
                       f"in {dt:.1f} s, host nproc={os.cpu_count()}")}
    return keys / dt / 1e9, info


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    threads = max(1, min(os.cpu_count() or 1, 64))
    n_sample = 4_000_000 if args.config != "c1" else 1_000_000
    steps = max(1, args.steps)
    per_step = max(1.0, min(args.cpu_seconds, 60.0 / steps))
    vals = []
    info = None
    for _ in range(steps):
        v, info = cpu_reference_run(n_sample, threads, per_step, args.config)
        vals.append(v)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup,
        # the workload's n at the measured rate (each step times a bounded sample of it)
        "ms_per_step": (args.n or {"c1": 10**6, "c5": 10**9}.get(args.config, 10**8)) / (value * 1e9) * 1e3,
        "sample_seconds_per_step": per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded SplitMix64, generator.cpp)",
        "config": {"workload": f"{args.config}: reference radix_sort_lsd on host cores (bounded samples)",
                   "algorithm": "radix", "keys_per_sample": n_sample},
        "cpu_baseline": dict(info, value=value, unit=UNIT),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- our arm
def profile_phases(lib):
    import ctypes as C

    ms = (C.c_float * 512)()
    names = C.create_string_buffer(512 * 16)
    cnt = C.c_int(0)
    na = C.c_int(0)
    rc = lib.isort_profile_end(ms, names, 16, 512, C.byref(cnt), C.byref(na))
    if rc:
        raise RuntimeError(lib.isort_last_error().decode())
    out = []
    for i in range(cnt.value):
        out.append((names.raw[i * 16:(i + 1) * 16].split(b"\0")[0].decode(), ms[i]))
    return out, na.value


def time_device_sort(sorter, keys, steps, warmup, lib, dist=None):
    """K timed steps (CUDA events on the sort's stream) for the value, then K more
    with per-kernel events between launches (isort_profile_*) for the phases and
    the roofline: the events add launch gaps, so they stay out of the value."""
    import torch

    for _ in range(warmup):
        sorter(keys)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = lib.isort_launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(steps):
        sorter(keys)
    end.record()
    torch.cuda.synchronize()
    launches = lib.isort_launch_count() - l0
    ms = start.elapsed_time(end) / steps
    lib.isort_profile_begin()
    for _ in range(steps):
        sorter(keys, eager=True)  # per-kernel events need the eager launch sequence
    torch.cuda.synchronize()
    phases, n_active = profile_phases(lib)
    if dist is not None:
        dist.barrier()
    return ms, phases, n_active, launches


def pass_stats(phases, steps, n_active):
    """Average duration of the executed one-sweep passes (ignore no-op slots)."""
    by = {}
    for name, ms in phases:
        by.setdefault(name, []).append(ms)
    passes = []
    for name, v in by.items():
        if name.startswith("pass"):
            passes.append((int(name[4:]), v))
    passes.sort()
    executed = [v for i, v in passes if i < n_active]
    flat = [x for v in executed for x in v]
    per_phase = {name: sum(v) / len(v) for name, v in by.items()}
    return (sum(flat) / len(flat) if flat else None), per_phase


def main_ours(args):
    import numpy as np
    import torch

    from paper_1206_3511_b200 import _lib, device, inputs

    world, rank, local = dist_env()
    dist = None
    if world > 1:
        import torch.distributed as tdist

        backend = os.environ.get("ISORT_DIST_BACKEND", "nccl")
        if backend == "nccl":
            torch.cuda.set_device(local)
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # plumbing check only (several ranks may share one GPU): gloo + CPU-staged exchange
            torch.cuda.set_device(local % torch.cuda.device_count())
            tdist.init_process_group(backend)
        dist = tdist
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    lib = _lib.load()
    peak, peak_src = measured_peak()

    n = args.n or {"c1": 10**6, "c5": 10**9 // max(world, 1)}.get(args.config, 10**8)
    cfg = args.config
    host_keys = inputs.config_keys(cfg, n, seed=42 + 7919 * rank if cfg not in ("c4a", "c4b") else 42)
    bound = inputs.config_range_bound(cfg)
    keys = torch.from_numpy(host_keys.view(np.int32)).to(dev)

    results = {}
    if world > 1:
        from paper_1206_3511_b200 import partition

        for alg in ("radix", "bucket"):
            ms, info = partition.bench_distributed(keys, alg, bound, args.steps, args.warmup, dist)
            results[alg] = {"ms": ms, "info": info}
    else:
        for alg in ("radix", "bucket"):
            use_graph = args.graph != "off"
            sorter = device.Sorter(n, 4, alg, None, range_bound=bound, device=dev, graph=use_graph)
            with ClockSampler(dev.index) as cs:
                ms, phases, n_active, launches = time_device_sort(sorter, keys, args.steps, args.warmup, lib)
            clocks = cs.summary()
            pavg, per_phase = pass_stats(phases, args.steps, n_active)
            # parity after timing (outside the timed region): sorted + same multiset
            out = sorter.keys_out
            ok_sorted = device.is_sorted_u32(out)
            ok_sum = int(out.to(torch.int64).bitwise_and(0xFFFFFFFF).sum()) == int(
                keys.to(torch.int64).bitwise_and(0xFFFFFFFF).sum())
            if use_graph:  # replays bypass the host launch counter: count the captured kernels
                launches = sorter.launches_per_call * args.steps
            results[alg] = {"ms": ms, "pass_ms": pavg, "n_active": n_active, "phases": per_phase,
                            "launches": launches, "clocks": clocks, "parity": bool(ok_sorted and ok_sum),
                            "graph": use_graph}
            del sorter
            torch.cuda.empty_cache()

    total_keys = n * world
    line = None
    if rank == 0:
        r = results["radix"]
        b = results["bucket"]
        value = total_keys / (r["ms"] / 1e3) / 1e9
        bvalue = total_keys / (b["ms"] / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32",
            "data": "synthetic: seeded SplitMix64 keys bit-identical to the reference generate() (inputs.py)",
            "config": {"workload": f"{cfg}: n={n:,} u32 keys per GPU, LSD radix sort (8-bit digits, "
                                   "one-sweep passes; trivial passes skipped)",
                       "n_per_gpu": n, "total_keys": total_keys, "algorithm": "radix",
                       "l2": "input+output 800 MB per GPU > 126 MB L2 (no flush needed)" if n >= 10**8 else
                             "input fits L2 (latency-bound config)",
                       "parallelism": f"key-range partition x{world}" if world > 1 else "single GPU",
                       "cuda_graph": bool(results["radix"].get("graph", False)) if world == 1 else False},
        }
        if world == 1:
            pass_bytes = 8 * n  # read 4n + write 4n per one-sweep pass (keys only)
            achieved = pass_bytes / (r["pass_ms"] / 1e3) / 1e9 if r["pass_ms"] else None
            traffic, traffic_src = ncu_traffic("k_onesweep") if n == N_DEFAULT else (None, None)
            line["roofline"] = {
                "bound": "hbm", "kernel": "k_onesweep<u32> (one digit pass)", "achieved": achieved,
                "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                "frac": achieved / peak if achieved else None, "traffic": traffic,
                "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": pass_bytes, "launch_ms": r["pass_ms"],
                "passes_executed": r["n_active"],
                "whole_sort_bytes": 4 * n + 8 * n * r["n_active"],
                "whole_sort_frac": (4 * n + 8 * n * r["n_active"]) / (r["ms"] / 1e3) / 1e9 / peak,
            }
            line["phases_ms"] = {k: round(v, 4) for k, v in r["phases"].items()}
            line["gpu_launches"] = r["launches"]
            line["clocks"] = r["clocks"]
            line["parity"] = {"radix": r["parity"], "bucket": b["parity"]}
            bb = 4 * n + 8 * n * b["n_active"] + 8 * n  # hist + passes + segment sort
            seg_ms = b["phases"].get("segments")
            seg_traffic, seg_src = ncu_traffic("k_bucket_segments") if n == N_DEFAULT else (None, None)
            seg_ach = 8 * n / (seg_ms / 1e3) / 1e9 if seg_ms else None
            line["bucket"] = {"value": bvalue, "ms_per_step": b["ms"], "passes_executed": b["n_active"],
                              "roofline": {"bound": "hbm", "kernel": "k_bucket_segments<u32> (in-smem sort of "
                                           "the super-buckets, in place)", "achieved": seg_ach, "peak": peak,
                                           "unit": "GB/s", "frac": seg_ach / peak if seg_ach else None,
                                           "traffic": seg_traffic, "traffic_source": seg_src,
                                           "algorithmic_bytes_per_launch": 8 * n, "launch_ms": seg_ms},
                              "phases_ms": {k: round(v, 4) for k, v in b["phases"].items()},
                              "whole_sort_bytes": bb, "whole_sort_frac": bb / (b["ms"] / 1e3) / 1e9 / peak,
                              "gpu_launches": b["launches"]}
        else:
            line["gpu_launches"] = r["info"].get("launches")
            line["phases_ms"] = r["info"].get("phases")
            line["exchange"] = r["info"].get("exchange")
            line["max_over_mean_received"] = r["info"].get("max_over_mean_received")
            line["bucket"] = {"value": bvalue, "ms_per_step": b["ms"], "phases_ms": b["info"].get("phases")}

    # ------------------------------------------------ e2e through the host C-ABI
    if not args.no_e2e:
        import numpy as np

        hin = torch.empty(n, dtype=torch.int32, pin_memory=True)
        hin.numpy()[:] = host_keys.view(np.int32)
        hout = torch.empty(n, dtype=torch.int32, pin_memory=True)
        e2e = {}
        d2h_bytes = 4 * n
        for alg in ("radix", "bucket"):
            if world == 1:
                def call():
                    if alg == "radix":
                        rc = lib.isort_radix_sort_host_u32(hin.data_ptr(), hout.data_ptr(), n, dev.index)
                    else:
                        rc = lib.isort_bucket_sort_host_u32(hin.data_ptr(), hout.data_ptr(), n, bound, dev.index)
                    _lib.check(rc)
            else:
                # the distributed sort end to end: this rank's shard H2D from pinned memory,
                # the key-range sort across the ranks, this rank's key range D2H
                from paper_1206_3511_b200 import partition

                sorter_e = partition.KeyRangeSorter(dist, partition.CudaOps(dev))
                if os.environ.get("ISORT_FUSED_EXCHANGE", "1") != "0":
                    partition.enable_fused(sorter_e, keys, alg)
                dkeys = torch.empty(n, dtype=torch.int32, device=dev)
                hout_e = torch.empty(int(1.5 * n) + (1 << 16), dtype=torch.int32, pin_memory=True)
                got = [0]

                def call():
                    dkeys.copy_(hin, non_blocking=True)
                    sk, _, _ = sorter_e.sort(dkeys, None, algorithm=alg)
                    m = sk.numel()
                    if m > hout_e.numel():
                        raise RuntimeError("received more keys than the pinned output buffer")
                    hout_e[:m].copy_(sk, non_blocking=True)
                    torch.cuda.current_stream(dev).synchronize()
                    got[0] = m

            for _ in range(max(1, args.warmup)):
                call()
            if dist is not None:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                call()
            dt = (time.perf_counter() - t0) / args.steps
            if dist is not None:
                t = torch.tensor([dt], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dt = float(t.item())
            if world > 1:
                d2h_bytes = 4 * got[0]
                if sorter_e.peers is not None:
                    sorter_e.peers.close()
            e2e[alg] = {"value": n * world / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": 4 * n,
                        "d2h_bytes_per_step": d2h_bytes, "ms_per_step": dt * 1e3,
                        "timer": "host perf_counter around the synchronous C-ABI call" if world == 1 else
                        "host perf_counter around shard H2D + distributed sort + own-range D2H, max over ranks"}
        if rank == 0:
            line["e2e"] = e2e["radix"]
            line["bucket"]["e2e"] = e2e["bucket"]

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = max(1, min(os.cpu_count() or 1, 64))
        v, info = cpu_reference_run(4_000_000 if n >= 4_000_000 else n, threads, args.cpu_seconds, cfg)
        line["cpu_baseline"] = dict(info, value=v, unit=UNIT)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return main_ours(args)


if __name__ == "__main__":
    sys.exit(main())
