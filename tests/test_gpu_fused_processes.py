"""The fused multi-GPU exchange across real processes: W ranks share the one
GPU gpurun provides, map each other's receive buffers through CUDA IPC, and run
counts -> partition-scatter into the peers' buffers -> local sort
(tools/two_rank_fused_check.py).  Host collectives go over gloo; no kernel of
one rank waits on a kernel of another.  Bit-exact against the global stable sort."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("n,world,algorithm", [(3_000_017, 2, "radix"), (1_000_003, 3, "radix"), (777, 2, "radix"),
                                               (12_000_001, 2, "radix"), (2_000_003, 3, "bucket")])
def test_fused_exchange_between_processes(n, world, algorithm):
    """bucket: each rank's local sort spreads its buckets over its own key range
    (isort_bucket_sort_span_u32); with the mixture keys the middle rank's range is
    the dense normal peak."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "two_rank_fused_check.py"), str(n), str(world),
                        algorithm],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "bit-exact=True" in r.stdout
