"""Checksums of the reference's output for every BASELINE.json configuration at
its stated size (test infrastructure; run where /root/reference was compiled):

    python tests/golden/make_full_size.py            # writes full_size_checksums.json

C1 (10^6 keys), C2, C3, C4a (10^8 keys) and C4b (C4a reversed, tags = positions) are sorted by the
UNMODIFIED reference (oracle/_ref/libintsort_ref.so): radix_sort_lsd at base 256
(proj/core/src/sort.cpp:112-119) and, as a cross-check, bucket_sort with the
config's range bound (sort.cpp:136-152); the two agree by construction (both are
the stable sort by key).  Inputs come from the reference's own generate()
(generator.cpp:115-156).  C5 (10^9-key mixture, a harness addition with no
reference generator) would need ~48 GB of host Records for the reference sort,
so it is sorted by the oracle's keys+positions restatement of the same LSD sort
(oracle/isort_oracle.c orc_radix_sort_u32), which tests/test_oracle.py pins to
the reference.

Each entry stores SHA-256 of: the input keys (u32 LE), the sorted keys (u32 LE),
and the stable positions (the output records' tags, u32 LE).  The GPU tests
(tests/test_gpu_full_size.py) and bench.py's parity check compare against these.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.binding import Oracle, Reference  # noqa: E402

U32_MAX = (1 << 32) - 1
OUT = os.path.join(HERE, "full_size_checksums.json")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).astype("<u4", copy=False).tobytes()).hexdigest()


def entry(keys_in, keys_out, pos_out, source, **extra):
    return dict(n=int(keys_in.size), input_sha256=sha(keys_in), sorted_keys_sha256=sha(keys_out),
                stable_positions_sha256=sha(pos_out), source=source, **extra)


def main(which=None) -> None:
    ref, orc = Reference(), Oracle()
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    sizes = {"c1": 1_000_000}  # the CPU-runnable config; the others are 10^8
    specs = {
        "c1": (1, U32_MAX),
        "c2": (1, U32_MAX),
        "c3": (1, 1023),
        "c4a": (2, U32_MAX),
        "c4b": (2, U32_MAX),
    }
    for name, (case_id, bound) in specs.items():
        if which and name not in which:
            continue
        t0 = time.time()
        n = sizes.get(name, 100_000_000)
        seq = ref.generate(case_id, n, bound, 42)
        if name == "c4b":
            seq = seq[::-1].copy()
            seq["tag"] = np.arange(n, dtype=np.uint64)
        out = ref.radix_sort_lsd(seq, 256)
        t_radix = time.time() - t0
        bk = ref.bucket_sort(seq, bound)
        agree = bool(np.array_equal(bk, out))
        assert agree, f"{name}: reference bucket_sort != radix_sort_lsd"
        res[name] = entry(seq["key"], out["key"], out["tag"],
                          "reference radix_sort_lsd(base 256) == bucket_sort(M) (oracle/_ref)",
                          range_bound=bound, generate=dict(case_id=case_id, n=n, range_bound=bound, seed=42,
                                                           reversed=name == "c4b"))
        print(f"{name}: {time.time() - t0:.1f} s (radix {t_radix:.1f} s)", flush=True)
        json.dump(res, open(OUT, "w"), indent=1)
        del seq, out, bk
    if not which or "c5" in which:
        t0 = time.time()
        n5 = 1_000_000_000
        k = orc.mixture_u32(n5, 42)
        ko, vo = orc.sort_u32(k, with_index=True)
        res["c5"] = entry(k, ko, vo, "oracle orc_radix_sort_u32 (keys + stable positions; pinned to the reference)",
                          range_bound=U32_MAX, generate=dict(mixture=True, n=n5, seed=42))
        print(f"c5: {time.time() - t0:.1f} s", flush=True)
        json.dump(res, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main(set(sys.argv[1:]) or None)
