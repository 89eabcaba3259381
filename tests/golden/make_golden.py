"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the build container, where /root/reference exists and
`make -C oracle ref` has produced oracle/_ref/libintsort_ref.so:

    python tests/golden/make_golden.py

Writes tests/golden/reference_vectors.npz (small seeded cases: inputs from the
reference's own generate(), outputs of its radix_sort_lsd / bucket_sort /
counting_sort_by_digit / build_radix_plan / bucket_index) and
tests/golden/reference_checksums.json (SHA-256 of the reference's sorted
output records for 10^6-key configuration-shaped inputs).  The GPU box has no
/root/reference; the tests read these fixtures instead.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.binding import RECORD_DTYPE, Oracle, Reference  # noqa: E402

U32_MAX = (1 << 32) - 1


def small_specs():
    """Seeded small specs over all six cases plus u32-range ones (make_golden's own stream)."""
    rng = np.random.default_rng(20121206)
    specs = []
    for case_id in range(1, 7):
        for n in (0, 1, 2, 7, 31, 32, 33, 255, 256, 257, 1000):
            specs.append(dict(case_id=case_id, n=n, range_bound=None, seed=int(rng.integers(1 << 62))))
    for n in (1, 5, 100, 1999, 4096, 7680, 7681):
        for bound in (U32_MAX, 1023, 1, 0, (1 << 40)):
            specs.append(dict(case_id=1, n=n, range_bound=bound, seed=int(rng.integers(1 << 62))))
    return specs


def main() -> None:
    ref = Reference()
    arrays = {}
    meta = []
    for i, sp in enumerate(small_specs()):
        seq = ref.generate(sp["case_id"], sp["n"], sp["range_bound"], sp["seed"])
        bound = sp["range_bound"] if sp["range_bound"] is not None else Oracle().default_range_bound(sp["case_id"])
        r10 = ref.radix_sort_lsd(seq, 10)
        r256 = ref.radix_sort_lsd(seq, 256)
        bk = ref.bucket_sort(seq, bound)
        digits10 = ref.build_radix_plan(seq, 10)
        cpass = ref.counting_sort_by_digit(seq, 10, digits10, digits10 - 1) if sp["n"] else seq
        arrays[f"in_{i}"] = seq["key"].copy()
        arrays[f"radix10_{i}"] = r10["tag"].astype(np.uint32)
        arrays[f"radix256_{i}"] = r256["tag"].astype(np.uint32)
        arrays[f"bucket_{i}"] = bk["tag"].astype(np.uint32)
        arrays[f"count_top_{i}"] = cpass["tag"].astype(np.uint32)
        meta.append(dict(sp, bound=bound, digits10=digits10, digits256=ref.build_radix_plan(seq, 256)))
    # bucket_index samples incl. the 2^72 corner (test_sort.cpp:168-174)
    bi_rng = np.random.default_rng(7)
    bidx = []
    for _ in range(2000):
        bound = int(bi_rng.integers(1, 1 << 40))
        count = int(bi_rng.integers(1, 1 << 32))
        key = int(bi_rng.integers(0, bound + 1))
        bidx.append((key, count, bound, ref.bucket_index(key, count, bound)))
    for key, count, bound in [((1 << 40), (1 << 32), (1 << 40)), (0, 1 << 32, 1 << 40), (U32_MAX, 10**8, U32_MAX),
                              (999, 10, 999), (500, 10, 999), (U32_MAX, 10**9, U32_MAX),
                              ((1 << 64) - 1, 3, (1 << 64) - 1), (12345, 10**8, (1 << 63) + 5)]:
        bidx.append((key, count, bound, ref.bucket_index(key, count, bound)))
    arrays["bucket_index"] = np.array(bidx, dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **arrays)
    with open(os.path.join(HERE, "reference_vectors.json"), "w") as f:
        json.dump(meta, f, indent=0)

    # checksums of the reference's output at 10^6 (config-shaped)
    orc = Oracle()
    n = 1_000_000
    checks = {}
    cases = {
        "u32_uniform": ref.generate(1, n, U32_MAX, 42),
        "u32_small_range_1023": ref.generate(1, n, 1023, 42),
        "u32_sorted": ref.generate(2, n, U32_MAX, 42),
    }
    rev = cases["u32_sorted"][::-1].copy()
    rev["tag"] = np.arange(n, dtype=np.uint64)
    cases["u32_reverse"] = rev
    mix = np.empty(n, dtype=RECORD_DTYPE)
    mix["key"] = orc.mixture_u32(n, 42)
    mix["tag"] = np.arange(n, dtype=np.uint64)
    cases["u32_mixture"] = mix
    for name, seq in cases.items():
        out_r = ref.radix_sort_lsd(seq, 256)
        out_b = ref.bucket_sort(seq, U32_MAX)
        assert (out_r == out_b).all()
        checks[name] = dict(
            n=n,
            input_sha256=hashlib.sha256(seq["key"].astype(np.uint32).tobytes()).hexdigest(),
            sorted_records_sha256=hashlib.sha256(out_r.tobytes()).hexdigest(),
        )
    with open(os.path.join(HERE, "reference_checksums.json"), "w") as f:
        json.dump(checks, f, indent=1)
    print(f"wrote {len(meta)} small cases, {len(bidx)} bucket_index samples, {len(checks)} checksums")

    # an ISRT sequence file written by the reference's own writer (sequence_io.cpp:63-70),
    # the file of its test_sequence_io.cpp:102-113 round trip (case 6, n = 500, seed 99),
    # plus a 2^40-range case-1 file: pins our reader and writer byte for byte
    seqs = {}
    for name, (case_id, n, bound, seed) in {"reference_case6.isrt": (6, 500, 1_000_000, 99),
                                            "reference_case1_2p40.isrt": (1, 3000, 1 << 40, 7)}.items():
        rec = ref.generate(case_id, n, bound if case_id == 1 else None, seed)
        ref.write_sequence_file(os.path.join(HERE, name), (case_id, 0, bound, seed), rec)
        seqs[name] = dict(case_id=case_id, n=n, range_bound=bound, seed=seed,
                          keys_sha256=hashlib.sha256(rec["key"].astype("<u8").tobytes()).hexdigest())
    with open(os.path.join(HERE, "reference_sequences.json"), "w") as f:
        json.dump(seqs, f, indent=1)


if __name__ == "__main__":
    main()
