"""Randomised check of the bulk-copy pass (k_onesweep_t): random sizes in [4M, 7M), random
distributions, radix / bucket, keys only / positions, u32 / u64, against numpy's stable sort.
    python tools/fuzz_tma.py [iterations] [seed]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1206_3511_b200 import device

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
bad = 0
for it in range(iters):
    n = int(rng.integers(4 << 20, 7 << 20))
    kb = 4 if rng.random() < 0.7 else 8
    alg = "radix" if kb == 8 or rng.random() < 0.5 else "bucket"
    vals = "iota" if rng.random() < 0.5 else None
    kind = rng.choice(["uniform", "few", "clustered", "runs", "bytes"])
    hi = (1 << 32) if kb == 4 else (1 << 63)
    dt = np.uint32 if kb == 4 else np.uint64
    if kind == "uniform":
        k = rng.integers(0, hi, size=n, dtype=np.uint64).astype(dt)
    elif kind == "few":
        k = rng.integers(0, int(rng.integers(5000, 200000)), size=n, dtype=np.uint64).astype(dt)
    elif kind == "clustered":
        c = rng.normal(hi / 2, hi / 4096, size=n)
        k = np.clip(c, 0, hi - 1).astype(np.uint64).astype(dt)
    elif kind == "runs":
        k = np.concatenate([np.sort(x) for x in np.array_split(rng.integers(0, hi, size=n, dtype=np.uint64).astype(dt),
                                                               int(rng.integers(3, 400)))])
    else:  # only some bytes vary
        m = int(rng.integers(1, 1 << (8 * kb - 1))) | 0xFF00
        k = (rng.integers(0, hi, size=n, dtype=np.uint64) & np.uint64(m)).astype(dt)
    t = torch.from_numpy(k.view(np.int32 if kb == 4 else np.int64).copy()).cuda()
    s = device.Sorter(n, kb, alg, vals, range_bound=(1 << 32) - 1 if kb == 4 else None)
    ko, vo = s(t)
    torch.cuda.synchronize()
    order = np.argsort(k, kind="stable")
    ok = np.array_equal(ko.cpu().numpy().view(dt), k[order])
    if vals:
        ok = ok and np.array_equal(vo.cpu().numpy().view(np.uint32), order.astype(np.uint32))
    bad += not ok
    print(f"{it:3d} n={n} u{8 * kb} {alg:6s} {'pairs' if vals else 'keys '} {kind:9s} {'ok' if ok else 'MISMATCH'}", flush=True)
print("mismatches:", bad)
sys.exit(1 if bad else 0)
