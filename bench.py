#!/usr/bin/env python
"""bench.py -- Gkeys/s sorting 100M uint32 keys (LSD radix & bucket) on B200.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` prints ONE
JSON line on rank 0.  A step = one full sort (one pass of the hot path) of the
configuration's keys.

N = 1: BASELINE.json configs[1] (C2: 10^8 u32 keys, uniform over [0, 2^32),
       seed 42 -- the reference's generate() keys), resident in HBM.
N > 1: one process per GPU (the driver's torchrun, or this script re-executing
       itself under torch.distributed.run when --gpus N > 1 is given without a
       WORLD_SIZE).  STRONG scaling of the same C2 job: rank r holds the r-th
       positional shard of the 10^8 keys, and the ranks sort them by key range
       (sampled splitters, fused partition -> peer-store exchange over
       NVLink/NVSwitch, or NCCL all-to-all; local sort; paper_1206_3511_b200/
       partition.py).  The C5 job (10^9-key mixture, sharded) is reported
       beside it in "c5".

value    = whole-job keys / device time (CUDA events on the sort's stream, max
           over ranks), inputs resident in HBM.  Headline: LSD radix; the bucket
           sort, the key+position ("pairs") sorts and C5 are extra objects.
parity   = SHA-256 of the sorted keys (and stable positions) against the
           reference's own output (tests/golden/full_size_checksums.json).
e2e      = the same metric through the host C-ABI call with host buffers
           (isort_radix_sort_host_u32: pinned keys H2D, sort, D2H); e2e_records =
           the reference's actual boundary, radix_sort_lsd(RecordSeq) via
           isort_radix_sort_records (16-byte records in and out).
roofline = the one-sweep digit pass (dominant kernel): 8n algorithmic bytes per
           launch / its live CUDA-event duration, against MEASURED_PEAKS.json.
cpu_baseline = the reference's own radix_sort_lsd (oracle/_ref, base 256, one
           thread -- the reference has no threading) on the full C2 input.
           `--impl reference` times exactly that, K times.
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
    p.add_argument("--config", default="c2", help="N = 1: c1 c2 c3 c4a c4b c5")
    p.add_argument("--n", type=int, default=None, help="total keys (default: the config's n)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-cpu-all-cores", action="store_true", help="reference arm: skip the all-cores aggregate")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-c5", action="store_true", help="N > 1: skip the sharded 10^9-key C5 job")
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


CONFIG_N = {"c1": 10**6, "c2": 10**8, "c3": 10**8, "c4a": 10**8, "c4b": 10**8, "c5": 10**9}
GENERATE = {"c1": (1, (1 << 32) - 1), "c2": (1, (1 << 32) - 1), "c3": (1, 1023), "c4a": (2, (1 << 32) - 1),
            "c4b": (2, (1 << 32) - 1)}


def checksums():
    try:
        with open(os.path.join(ROOT, "tests", "golden", "full_size_checksums.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def sha_u32(a) -> str:
    import hashlib

    import numpy as np

    return hashlib.sha256(np.ascontiguousarray(a).astype("<u4", copy=False).tobytes()).hexdigest()


# --------------------------------------------------------- reference arm
def reference_records(cfg: str, n: int):
    """The configuration's input as the reference's 16-byte Records, from the
    reference's own generate() (C4b: C4a reversed, tags = positions)."""
    import numpy as np

    from oracle.binding import RECORD_DTYPE, Oracle, Reference

    if cfg in GENERATE:
        case_id, bound = GENERATE[cfg]
        gen = Reference() if Reference.available() else Oracle()
        seq = gen.generate(case_id, n, bound, 42)
        if cfg == "c4b":
            seq = seq[::-1].copy()
            seq["tag"] = np.arange(n, dtype=np.uint64)
        return seq
    from paper_1206_3511_b200 import inputs

    seq = np.empty(n, dtype=RECORD_DTYPE)
    seq["key"] = inputs.config_keys(cfg, n)
    seq["tag"] = np.arange(n, dtype=np.uint64)
    return seq


def cpu_reference_sorts(seq, steps: int, warmup: int):
    """`steps` timed calls of the reference's radix_sort_lsd(seq, 256) on one host
    thread (ref_time_one: the region time_sort times, bench.cpp:81-84); warm-up
    calls on a 10^6-record prefix.  Returns (seconds per sort, kind)."""
    from oracle.binding import Oracle, Reference

    kind = "reference" if Reference.available() else "port"
    impl = Reference() if kind == "reference" else Oracle()
    for _ in range(warmup):
        if kind == "reference":
            impl.time_one("radix", seq[: min(seq.size, 10**6)], 0, 256)
        else:
            impl.radix_sort_lsd(seq[: min(seq.size, 10**6)], 256)
    times = []
    for _ in range(steps):
        if kind == "reference":
            times.append(impl.time_one("radix", seq, 0, 256))
        else:
            t0 = time.perf_counter()
            impl.radix_sort_lsd(seq, 256)
            times.append(time.perf_counter() - t0)
    return times, kind


def cpu_all_cores(cfg: str, target_s: float = 8.0, n_sample: int = 4_000_000):
    """Aggregate throughput of the reference radix_sort_lsd with every host core
    sorting its own seeded n_sample-record sample of the configuration
    concurrently (a separate figure: one reference sort cannot use more than one
    thread)."""
    import numpy as np

    from oracle.binding import RECORD_DTYPE, Oracle, Reference
    from paper_1206_3511_b200 import inputs

    threads = max(1, min(os.cpu_count() or 1, 64))
    impl = Reference() if Reference.available() else Oracle()
    samples = []
    for t in range(threads):
        seq = np.empty(n_sample, dtype=RECORD_DTYPE)
        seq["key"] = inputs.uniform_u32(n_sample, 42, start=t * n_sample).astype(np.uint64)
        seq["tag"] = np.arange(n_sample, dtype=np.uint64)
        samples.append(seq)
    counts = [0] * threads
    stop_at = time.perf_counter() + target_s

    def worker(i):
        while True:
            impl.radix_sort_lsd(samples[i], 256)  # ctypes releases the GIL
            counts[i] += 1
            if time.perf_counter() >= stop_at:
                break

    t0 = time.perf_counter()
    ths = [threading.Thread(target=worker, args=(i,)) for i in range(threads)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    dt = time.perf_counter() - t0
    return {"value": sum(counts) * n_sample / dt / 1e9, "unit": UNIT, "cores": threads,
            "sample": f"{threads} threads each sorting its own {n_sample:,}-record uniform u32 sample "
                      f"(reference radix_sort_lsd base 256), {sum(counts)} sorts in {dt:.1f} s"}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = args.config
    n = args.n or CONFIG_N[cfg]
    bounded = n > 2 * 10**8  # C5: the reference would need ~48 GB of host Records; a 10^8 sample stands in
    n_run = 10**8 if bounded else n
    seq = reference_records(cfg, n_run)
    steps = max(1, args.steps)
    times, kind = cpu_reference_sorts(seq, steps, args.warmup)
    sec = sum(times) / len(times)
    value = n_run / sec / 1e9
    sample = (f"reference radix_sort_lsd(RecordSeq, base 256) on one host thread, {n_run:,} {cfg} Records "
              f"(generate(), seed 42), {steps} timed sorts, median {statistics.median(times):.2f} s; "
              f"host nproc={os.cpu_count()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic: the reference's own generate() (SplitMix64, seed 42)",
        "config": {"workload": f"{cfg}: radix_sort_lsd of n={n_run:,} Records on the host (the reference is "
                               "single-threaded; it has no GPU or multi-GPU path)",
                   "n": n_run, "algorithm": "radix (base 256: 8-bit digits, 4 passes)",
                   "same_config": n_run == CONFIG_N[cfg], "step": "one full sort of the configuration's input"},
        "cpu_baseline": {"kind": kind, "cores": 1, "sample": sample, "value": value, "unit": UNIT},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_cpu_all_cores:
        line["cpu_all_cores"] = cpu_all_cores(cfg)
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


def time_device_sort(sorter, keys, steps, warmup, lib, profile=True):
    """K timed steps (CUDA events on the sort's stream) for the value, then K more
    with per-kernel events between launches (isort_profile_*) for the phases and
    the roofline: the events add launch gaps, so they stay out of the value."""
    import torch

    for _ in range(warmup):
        sorter(keys)
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
    phases, n_active = [], 0
    if profile:
        lib.isort_profile_begin()
        for _ in range(steps):
            sorter(keys, eager=True)  # per-kernel events need the eager launch sequence
        torch.cuda.synchronize()
        phases, n_active = profile_phases(lib)
    return ms, phases, n_active, launches


def pass_stats(phases, n_active):
    """Average duration of the executed one-sweep passes (ignore no-op slots)."""
    by = {}
    for name, ms in phases:
        by.setdefault(name, []).append(ms)
    passes = sorted((int(name[4:]), v) for name, v in by.items() if name.startswith("pass"))
    flat = [x for i, v in passes if i < n_active for x in v]
    per_phase = {name: sum(v) / len(v) for name, v in by.items()}
    return (sum(flat) / len(flat) if flat else None), per_phase


def one_gpu(args, lib, dev, peak, peak_src):
    import numpy as np
    import torch

    from paper_1206_3511_b200 import _lib, device, inputs

    cfg = args.config
    n = args.n or CONFIG_N[cfg]
    host_keys = inputs.config_keys(cfg, n)
    bound = inputs.config_range_bound(cfg)
    chk = checksums().get(cfg) if n == CONFIG_N[cfg] else None
    input_pinned = chk is not None and sha_u32(host_keys) == chk["input_sha256"]
    keys = torch.from_numpy(host_keys.view(np.int32)).to(dev)
    use_graph = args.graph != "off"
    res, parity = {}, {}
    for alg in ("radix", "bucket"):
        for vals in (None, "iota"):
            tag = alg + ("_pairs" if vals else "")
            sorter = device.Sorter(n, 4, alg, vals, range_bound=bound, device=dev, graph=use_graph)
            with ClockSampler(dev.index) as cs:
                ms, phases, n_active, launches = time_device_sort(sorter, keys, args.steps, args.warmup, lib,
                                                                  profile=True)
            pavg, per_phase = pass_stats(phases, n_active)
            if use_graph:  # replays bypass the host launch counter: count the captured kernels
                launches = sorter.launches_per_call * args.steps
            res[tag] = {"ms": ms, "pass_ms": pavg, "n_active": n_active, "phases": per_phase, "launches": launches,
                        "clocks": cs.summary()}
            # parity after timing (outside the timed region): the reference's own output digests
            out_k = sorter.keys_out.cpu().numpy().view(np.uint32)
            if input_pinned:
                ok = sha_u32(out_k) == chk["sorted_keys_sha256"]
                if vals:
                    ok = ok and sha_u32(sorter.vals_out.cpu().numpy().view(np.uint32)) == \
                        chk["stable_positions_sha256"]
                parity[tag] = bool(ok)
            else:
                parity[tag] = bool(device.is_sorted_u32(sorter.keys_out)) and "unpinned (sorted only)"
            del sorter
            torch.cuda.empty_cache()
    return n, host_keys, bound, res, parity, input_pinned


def e2e_keys(lib, host_keys, n, bound, steps, warmup, dev):
    import numpy as np
    import torch

    from paper_1206_3511_b200 import _lib

    hin = torch.empty(n, dtype=torch.int32, pin_memory=True)
    hin.numpy()[:] = host_keys.view(np.int32)
    hout = torch.empty(n, dtype=torch.int32, pin_memory=True)
    out = {}
    for alg in ("radix", "bucket"):
        def call():
            if alg == "radix":
                rc = lib.isort_radix_sort_host_u32(hin.data_ptr(), hout.data_ptr(), n, dev.index)
            else:
                rc = lib.isort_bucket_sort_host_u32(hin.data_ptr(), hout.data_ptr(), n, bound, dev.index)
            _lib.check(rc)

        for _ in range(max(1, warmup)):
            call()
        t0 = time.perf_counter()
        for _ in range(steps):
            call()
        dt = (time.perf_counter() - t0) / steps
        out[alg] = {"value": n / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n,
                    "ms_per_step": dt * 1e3, "timer": "host perf_counter around the synchronous C-ABI call "
                                                      "(pinned host keys in and out)"}
    return out


def e2e_records(cfg, n, steps, warmup, dev, chk):
    """radix_sort_lsd(RecordSeq) at the reference's own boundary: 16-byte host
    records in, sorted records out (isort_radix_sort_records: H2D, pack, key +
    position sort, gather, D2H)."""
    import numpy as np

    import paper_1206_3511_b200 as isort

    seq = reference_records_product(cfg, n)
    for _ in range(max(1, warmup)):
        out = isort.radix_sort_lsd(seq, 256)
    t0 = time.perf_counter()
    for _ in range(steps):
        out = isort.radix_sort_lsd(seq, 256)
    dt = (time.perf_counter() - t0) / steps
    ok = None
    if chk is not None:
        ok = sha_u32(out["key"]) == chk["sorted_keys_sha256"] and sha_u32(out["tag"]) == chk["stable_positions_sha256"]
    return {"value": n / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 16 * n,
            "ms_per_step": dt * 1e3, "parity": ok,
            "timer": "host perf_counter around intsort.radix_sort_lsd(seq, 256) (pageable 16-byte Records)"}


def reference_records_product(cfg, n):
    """Records of the configuration built by the product's input module (no oracle)."""
    import numpy as np

    from paper_1206_3511_b200 import inputs
    from paper_1206_3511_b200.intsort import RECORD_DTYPE

    seq = np.empty(n, dtype=RECORD_DTYPE)
    seq["key"] = inputs.config_keys(cfg, n)
    seq["tag"] = np.arange(n, dtype=np.uint64)
    return seq


def gather_to_rank0(dist, t, dev):
    """Concatenate every rank's 1-D int32 tensor on rank 0 (rank order); None elsewhere."""
    import torch

    world, rank = dist.get_world_size(), dist.get_rank()
    if dist.get_backend() == "gloo":  # gloo's point-to-point moves host memory only
        dev = torch.device("cpu")
        t = t.cpu()
    size = torch.tensor([t.numel()], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(size) for _ in range(world)]
    dist.all_gather(sizes, size)
    sizes = [int(x.item()) for x in sizes]
    if rank == 0:
        parts = [t]
        for r in range(1, world):
            buf = torch.empty(sizes[r], dtype=t.dtype, device=dev)
            if sizes[r]:
                dist.recv(buf, src=r)
            parts.append(buf)
        return torch.cat(parts)
    if t.numel():
        dist.send(t.contiguous(), dst=0)
    return None


def multi_gpu(args, lib, dev, dist, world, rank):
    import numpy as np
    import torch

    from paper_1206_3511_b200 import inputs, partition

    res = {}
    jobs = [("c2", args.n or CONFIG_N["c2"])]
    if not args.no_c5:
        jobs.append(("c5", CONFIG_N["c5"]))
    sums = checksums()
    for cfg, n_total in jobs:
        shard = inputs.config_shard(cfg, n_total, rank, world)
        keys = torch.from_numpy(shard.view(np.int32)).to(dev)
        bound = inputs.config_range_bound(cfg)
        for alg in (("radix", "bucket") if cfg == "c2" else ("radix",)):
            with ClockSampler(dev.index) as cs:
                ms, info, sk = partition.bench_distributed(keys, alg, bound, args.steps, args.warmup, dist)
            full = gather_to_rank0(dist, sk, dev)
            ok = None
            if rank == 0 and n_total == CONFIG_N[cfg] and cfg in sums:
                ok = sha_u32(full.cpu().numpy().view(np.uint32)) == sums[cfg]["sorted_keys_sha256"]
            res[(cfg, alg)] = {"ms": ms, "info": info, "n": n_total, "parity": ok, "clocks": cs.summary()}
            del sk, full
            torch.cuda.empty_cache()
        del keys
    return res


def relaunch(args):
    """--gpus N without a torchrun environment: run this script as N ranks."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main_ours(args):
    import numpy as np
    import torch

    from paper_1206_3511_b200 import _lib

    world, rank, local = dist_env()
    dist = None
    plumbing = False
    if world > 1:
        import torch.distributed as tdist

        ngpu = torch.cuda.device_count()
        backend = os.environ.get("ISORT_DIST_BACKEND", "nccl" if ngpu >= world else "gloo")
        if backend == "nccl":
            torch.cuda.set_device(local)
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # plumbing check only (ranks share a GPU): host collectives over gloo
            plumbing = True
            torch.cuda.set_device(local % ngpu)
            tdist.init_process_group("gloo")
        dist = tdist
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    lib = _lib.load()
    _lib.check(lib.isort_init(dev.index))
    peak, peak_src = measured_peak()

    line = None
    if world == 1:
        n, host_keys, bound, res, parity, pinned = one_gpu(args, lib, dev, peak, peak_src)
        r, b = res["radix"], res["bucket"]
        value = n / (r["ms"] / 1e3) / 1e9
        pass_bytes = 8 * n  # read 4n + write 4n per one-sweep pass (keys only)
        achieved = pass_bytes / (r["pass_ms"] / 1e3) / 1e9 if r["pass_ms"] else None
        traffic, traffic_src = ncu_traffic("k_onesweep_t") if n == N_DEFAULT else (None, None)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32",
            "data": "synthetic: seeded SplitMix64 keys bit-identical to the reference generate() (inputs.py)",
            "config": {"workload": f"{args.config}: n={n:,} u32 keys, LSD radix sort (8-bit digits, one-sweep "
                                   "passes; trivial passes skipped), keys resident in HBM",
                       "n": n, "algorithm": "radix",
                       "l2": "input+output 800 MB > 126 MB L2 (no flush needed)" if n >= 10**8 else
                             "input fits L2 (latency-bound config)",
                       "parallelism": "single GPU", "cuda_graph": args.graph != "off"},
            "roofline": {
                "bound": "hbm", "kernel": ("k_onesweep_t<u32> (one digit pass, bulk-copy write-out)" if n >= (4 << 20) else
                                             "k_onesweep<u32> (one digit pass, small-input tile)"), "achieved": achieved,
                "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                "frac": achieved / peak if achieved else None, "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": pass_bytes, "launch_ms": r["pass_ms"],
                "passes_executed": r["n_active"], "whole_sort_bytes": 4 * n + 8 * n * r["n_active"],
                "whole_sort_frac": (4 * n + 8 * n * r["n_active"]) / (r["ms"] / 1e3) / 1e9 / peak},
            "phases_ms": {k: round(v, 4) for k, v in r["phases"].items()},
            "gpu_launches": r["launches"], "clocks": r["clocks"],
            "parity": dict(parity, reference="tests/golden/full_size_checksums.json (reference output SHA-256)"
                           if pinned else "input not pinned: sortedness only"),
        }
        bb = 4 * n + 8 * n * b["n_active"] + 8 * n  # hist + passes + segment sort
        seg_ms = b["phases"].get("segments")
        seg_traffic, seg_src = ncu_traffic("k_bucket_segments") if n == N_DEFAULT else (None, None)
        seg_ach = 8 * n / (seg_ms / 1e3) / 1e9 if seg_ms else None
        line["bucket"] = {"value": n / (b["ms"] / 1e3) / 1e9, "ms_per_step": b["ms"],
                          "passes_executed": b["n_active"],
                          "roofline": {"bound": "hbm", "kernel": "k_bucket_segments<u32> (in-smem sort of the "
                                       "super-buckets, in place)", "achieved": seg_ach, "peak": peak,
                                       "unit": "GB/s", "frac": seg_ach / peak if seg_ach else None,
                                       "traffic": seg_traffic, "traffic_source": seg_src,
                                       "algorithmic_bytes_per_launch": 8 * n, "launch_ms": seg_ms},
                          "phases_ms": {k: round(v, 4) for k, v in b["phases"].items()},
                          "whole_sort_bytes": bb, "whole_sort_frac": bb / (b["ms"] / 1e3) / 1e9 / peak,
                          "gpu_launches": b["launches"]}
        line["pairs"] = {
            alg: {"value": n / (res[alg + "_pairs"]["ms"] / 1e3) / 1e9, "ms_per_step": res[alg + "_pairs"]["ms"],
                  "unit": UNIT, "what": "u32 key + u32 stable position payload (generated on the device)",
                  "phases_ms": {k: round(v, 4) for k, v in res[alg + "_pairs"]["phases"].items()}}
            for alg in ("radix", "bucket")}
        if not args.no_e2e:
            e2e = e2e_keys(lib, host_keys, n, bound, args.steps, args.warmup, dev)
            line["e2e"] = e2e["radix"]
            line["bucket"]["e2e"] = e2e["bucket"]
            chk = checksums().get(args.config) if pinned else None
            line["e2e_records"] = e2e_records(args.config, n, max(1, min(args.steps, 10)), 1, dev, chk)
        if not args.no_cpu_baseline:
            seq = reference_records(args.config, n if n <= 2 * 10**8 else 10**8)
            times, kind = cpu_reference_sorts(seq, 1, 0)
            line["cpu_baseline"] = {"kind": kind, "cores": 1, "value": seq.size / times[0] / 1e9, "unit": UNIT,
                                    "sample": f"one reference radix_sort_lsd(base 256) of the full {seq.size:,}-"
                                              f"record {args.config} input on one host thread: {times[0]:.2f} s "
                                              f"(host nproc={os.cpu_count()})"}
    else:
        res = multi_gpu(args, lib, dev, dist, world, rank)
        if rank == 0:
            r, b = res[("c2", "radix")], res[("c2", "bucket")]
            n = r["n"]
            line = {
                "metric": METRIC, "value": n / (r["ms"] / 1e3) / 1e9, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u32",
                "data": "synthetic: seeded SplitMix64 keys bit-identical to the reference generate() (inputs.py)",
                "config": {"workload": f"c2: n={n:,} u32 keys in total, rank r holds the r-th positional shard; "
                                       "distributed LSD radix sort by key range",
                           "n": n, "n_per_gpu": n // world, "algorithm": "radix",
                           "parallelism": f"key-range partition x{world}",
                           "exchange": r["info"]["exchange"],
                           "plumbing_only": plumbing and "ranks share one GPU (gloo host collectives)"},
                "phases_ms": r["info"]["phases_ms"], "max_over_mean_received": r["info"]["max_over_mean_received"],
                "gpu_launches": r["info"]["launches"], "clocks": r["clocks"],
                "parity": {"radix": r["parity"], "bucket": b["parity"],
                           "reference": "rank-ordered concatenation vs the reference's sorted-keys SHA-256"},
                "bucket": {"value": n / (b["ms"] / 1e3) / 1e9, "ms_per_step": b["ms"],
                           "phases_ms": b["info"]["phases_ms"],
                           "max_over_mean_received": b["info"]["max_over_mean_received"]},
            }
            if ("c5", "radix") in res:
                c5 = res[("c5", "radix")]
                line["c5"] = {"value": c5["n"] / (c5["ms"] / 1e3) / 1e9, "unit": UNIT, "ms_per_step": c5["ms"],
                              "n": c5["n"], "n_per_gpu": c5["n"] // world, "phases_ms": c5["info"]["phases_ms"],
                              "max_over_mean_received": c5["info"]["max_over_mean_received"],
                              "exchange": c5["info"]["exchange"], "parity": c5["parity"]}
        if not args.no_e2e:
            e2e = distributed_e2e(args, lib, dev, dist, world, rank)
            if rank == 0:
                line["e2e"] = e2e
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def distributed_e2e(args, lib, dev, dist, world, rank):
    """The distributed sort end to end: this rank's shard H2D from pinned memory,
    the key-range sort, this rank's key range D2H; max over ranks."""
    import numpy as np
    import torch

    from paper_1206_3511_b200 import inputs, partition

    n_total = args.n or CONFIG_N["c2"]
    shard = inputs.config_shard("c2", n_total, rank, world)
    n = shard.size
    hin = torch.empty(n, dtype=torch.int32, pin_memory=True)
    hin.numpy()[:] = shard.view(np.int32)
    sorter = partition.KeyRangeSorter(dist, partition.CudaOps(dev))
    dkeys = torch.empty(n, dtype=torch.int32, device=dev)
    dkeys.copy_(hin)
    try:
        if os.environ.get("ISORT_FUSED_EXCHANGE", "1") != "0":
            partition.enable_fused(sorter, dkeys, "radix")
        hout = torch.empty(int(1.5 * n) + (1 << 16), dtype=torch.int32, pin_memory=True)
        got = [0]

        def call():
            dkeys.copy_(hin, non_blocking=True)
            sk, _, _ = sorter.sort(dkeys, None, algorithm="radix")
            m = sk.numel()
            if m > hout.numel():
                raise RuntimeError("received more keys than the pinned output buffer")
            hout[:m].copy_(sk, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
            got[0] = m

        for _ in range(max(1, args.warmup)):
            call()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            call()
        dt = (time.perf_counter() - t0) / args.steps
        t = torch.tensor([dt], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
        d2h = torch.tensor([got[0]], dtype=torch.int64, device=dev)
        dist.all_reduce(d2h, op=dist.ReduceOp.MAX)
    finally:
        if sorter.peers is not None:
            sorter.peers.close()
    return {"value": n_total / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": 4 * n,
            "d2h_bytes_per_step": 4 * int(d2h.item()), "ms_per_step": dt * 1e3,
            "timer": "host perf_counter around shard H2D + distributed sort + own-range D2H, max over ranks"}


def main():
    args = parse_args()
    world, _, _ = dist_env()
    if args.impl == "reference":
        return run_reference(args)
    if world == 1 and args.gpus > 1:
        return relaunch(args)
    return main_ours(args)


if __name__ == "__main__":
    sys.exit(main())
