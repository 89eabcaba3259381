"""Quick device-resident timing matrix (not the bench): radix / bucket, keys-only
and pairs, over several key ranges / bounds, CUDA events, median of reps.

    python tools/time_sorts.py [n] [reps]

Each case prints ms and Gkeys/s, and checks the output against numpy (keys) /
a stable argsort (positions) on a 1e6-key prefix-sized run first.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1206_3511_b200 import device, inputs  # noqa: E402


def keys_for(n, kind, seed=42):
    rng = np.random.default_rng(seed)
    if kind == "u32":
        return inputs.uniform_u32(n, seed)
    if kind.startswith("below:"):
        b = int(kind.split(":")[1])
        return rng.integers(0, b + 1, size=n, dtype=np.uint64).astype(np.uint32)
    if kind == "sorted":
        return np.sort(inputs.uniform_u32(n, seed))
    if kind == "reverse":
        return np.sort(inputs.uniform_u32(n, seed))[::-1].copy()
    if kind == "mixture":
        return inputs.config_keys("c5", n)
    raise ValueError(kind)


def time_case(n, kind, alg, vals, bound, reps, check=True):
    k = keys_for(n, kind)
    t = torch.from_numpy(k.view(np.int32)).cuda()
    s = device.Sorter(n, 4, alg, vals, range_bound=bound, graph=True)
    for _ in range(3):
        s(t)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s(t)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    ok = None
    if check:
        got = s.keys_out.cpu().numpy().view(np.uint32)
        order = np.argsort(k, kind="stable")
        ok = bool(np.array_equal(got, k[order]))
        if vals:
            ok = ok and bool(np.array_equal(s.vals_out.cpu().numpy().view(np.uint32), order.astype(np.uint32)))
    return ms, ok


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    cases = [("u32", None), ("below:1023", 1023), ("below:999999", 999_999), ("below:99999999", 99_999_999),
             ("below:4000000000", 4_000_000_000), ("sorted", None), ("reverse", None), ("mixture", None)]
    only = os.environ.get("TS_ONLY")
    for kind, bound in cases:
        if only and not any(o in kind for o in only.split(",")):
            continue
        for alg in ("radix", "bucket"):
            for vals in (None, "iota"):
                b = bound if bound is not None else (1 << 32) - 1
                ms, ok = time_case(n, kind, alg, vals, b, reps)
                print(f"{kind:18s} {alg:6s} {'pairs' if vals else 'keys ':5s} {ms:8.4f} ms "
                      f"{n / ms / 1e6:8.1f} Gkeys/s  ok={ok}", flush=True)


if __name__ == "__main__":
    main()
