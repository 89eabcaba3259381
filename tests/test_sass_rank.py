"""The one-sweep rank's stability rests on one instruction: a returning shared
atomic add (SASS ATOMS.ADD with a destination register; the non-returning counts
compile to ATOMS.POPC.INC.32 RZ) whose same-address lanes are granted in
ascending lane order.  k_selftest_atomic_order re-checks that property at load time, so it
must exercise the SAME instruction the rank compiles to.  This CPU test
disassembles libisort.so (cuobjdump) and pins:
  * the fast passes (SAFE = false; k_onesweep_t and k_onesweep) rank with ATOMS.ADD and have no MATCH,
  * the load-time self-test uses ATOMS.ADD (and MATCH.ANY as its reference),
  * the fallback pass (SAFE = true) ranks with MATCH.ANY,
  * the segment sort of the bucket path ranks with ATOMS.ADD too."""
from __future__ import annotations

import collections
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1206_3511_b200", "libisort.so")


@pytest.fixture(scope="module")
def sass_ops():
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "-sass", LIB], capture_output=True, text=True, check=True).stdout
    ops = collections.defaultdict(collections.Counter)
    fn = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"\b(ATOMS\.[A-Z0-9.]+|MATCH\.[A-Z]+)\s+(\w+)", line)
        if m and fn:
            op = m.group(1)
            if op.startswith("ATOMS") and m.group(2) != "RZ":
                op += ".RET"  # returns the old value: a rank, not a count
            ops[fn][op] += 1
    return ops


def _find(ops, *parts):
    hits = [f for f in ops if all(p in f for p in parts)]
    assert hits, f"no kernel matching {parts}"
    return hits


def _assert_fast(sass_ops, f):
    c = sass_ops[f]
    assert c["ATOMS.ADD.RET"] > 0, (f, dict(c))
    assert not any(k.startswith("MATCH") for k in c), f
    assert not any(k.endswith(".RET") and k != "ATOMS.ADD.RET" for k in c), (f, dict(c))


def test_fast_rank_is_returning_shared_atomic(sass_ops):
    # the rank is a returning ATOMS.ADD; the counts are non-returning (ATOMS.POPC.INC.32 RZ / ATOMS.ADD RZ)
    # k_onesweep_t<u32, RadixDigitizer<u32>, 512, 32, VALS=0, SAFE=0, LW>: keys-only passes over large inputs
    for f in _find(sass_ops, "k_onesweep_tIj", "RadixDigitizerIj", "Li512ELi32ELb0ELb0E"):
        _assert_fast(sass_ops, f)
    # k_onesweep_t<u32, RadixDigitizer<u32>, 512, 16, VALS=1, SAFE=0, LW>: the same with a payload
    for f in _find(sass_ops, "k_onesweep_tIj", "RadixDigitizerIj", "Li512ELi16ELb1ELb0E"):
        _assert_fast(sass_ops, f)
    # k_onesweep<u32, RadixDigitizer<u32>, 512, IPT, 1, VALS, SAFE=0, SCATTER=0, LW>: small inputs
    for f in _find(sass_ops, "k_onesweepIj", "RadixDigitizerIj", "Li512ELi16ELi1ELb0ELb0ELb0E"):
        _assert_fast(sass_ops, f)
    for f in _find(sass_ops, "k_onesweepIj", "RadixDigitizerIj", "Li512ELi12ELi1ELb1ELb0ELb0E"):
        _assert_fast(sass_ops, f)


def test_selftest_checks_the_same_instruction(sass_ops):
    # both rank forms (plain +1, and the segment sort's 16-bit packed increment) as
    # returning ATOMS.ADD, against MATCH.ANY
    for f in _find(sass_ops, "k_selftest_atomic_order"):
        assert sass_ops[f]["ATOMS.ADD.RET"] >= 2 and sass_ops[f]["MATCH.ANY"] > 0, (f, dict(sass_ops[f]))


def test_safe_rank_uses_match(sass_ops):
    for f in _find(sass_ops, "k_onesweep_tIj", "RadixDigitizerIj", "Li512ELi32ELb0ELb1E"):
        assert sass_ops[f]["MATCH.ANY"] > 0, f
    for f in _find(sass_ops, "k_onesweep_tIj", "RadixDigitizerIj", "Li512ELi16ELb1ELb1E"):
        assert sass_ops[f]["MATCH.ANY"] > 0, f
    for f in _find(sass_ops, "k_onesweepIj", "RadixDigitizerIj", "Li512ELi12ELi1ELb1ELb1ELb0E"):
        assert sass_ops[f]["MATCH.ANY"] > 0, f


def test_segment_sort_rank(sass_ops):
    for f in _find(sass_ops, "k_bucket_segments"):
        assert sass_ops[f]["ATOMS.ADD.RET"] > 0, f
