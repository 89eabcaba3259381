"""The fallback for a device whose same-address shared atomics were not granted
in lane order (k_selftest_atomic_order): ISORT_FORCE_SAFE_RANK=1 forces it, and
both sorts must stay bit-exact (radix: the __match_any_sync rank; bucket: the
radix pipeline finishes the bucket-grouped keys instead of the segment sort)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np, torch, sys
sys.path.insert(0, %r)
from paper_1206_3511_b200 import _lib, device
assert _lib.load().isort_rank_mode() == 0, "fallback not active"
rng = np.random.default_rng(3)
for n in (1, 5000, 24577, 1_000_003, 6_000_011):
    for alg in ("radix", "bucket"):
        for payload in (None, "iota"):
            k = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
            if n > 2:
                k[: n // 3] = k[0]  # duplicates: stability is observable
            s = device.Sorter(n, 4, alg, payload, range_bound=(1 << 32) - 1, graph=True)
            ko, vo = s(torch.from_numpy(k.view(np.int32)).cuda())
            torch.cuda.synchronize()
            order = np.argsort(k, kind="stable")
            assert np.array_equal(ko.cpu().numpy().view(np.uint32), k[order]), (n, alg, payload)
            if payload:
                assert np.array_equal(vo.cpu().numpy().view(np.uint32), order.astype(np.uint32)), (n, alg)
print("safe-rank ok")
""" % ROOT


@pytest.mark.gpu
def test_safe_rank_fallback_is_bit_exact():
    env = dict(os.environ, ISORT_FORCE_SAFE_RANK="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0 and "safe-rank ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
