"""The multi-GPU key-range protocol (paper_1206_3511_b200/partition.py) over
gloo with world_size 2 and 3 on CPU.  The per-rank kernels are replaced by a
torch-CPU stand-in with the same contract (stable partition by destination,
stable local sort) -- this tests the distributed logic: sampling, splitters,
count exchange, all-to-all-v, source-order stability and the rank-ordered
concatenation.  The CUDA kernels themselves are covered by the -m gpu tests."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1206_3511_b200.partition import KeyRangeSorter


def _u(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.int64) & 0xFFFFFFFF


class TorchCpuOps:
    """Stand-in for CudaOps on CPU tensors (test double, not a product path)."""

    def sample(self, keys, s):  # CudaOps.sample's contract: exactly s keys
        n = keys.numel()
        if n == 0:
            return torch.full((s,), -1, dtype=keys.dtype)
        return keys[(torch.arange(s, dtype=torch.int64) * n) // s].contiguous()

    def sort(self, keys):
        return keys[torch.sort(_u(keys), stable=True).indices]

    def partition(self, keys, vals, splitters, parts):
        k = _u(keys)
        dest = torch.zeros_like(k)
        for s in splitters:
            dest += (k >= s).to(torch.int64)
        order = torch.sort(dest, stable=True).indices
        counts = torch.bincount(dest, minlength=parts).to(torch.int64)
        return keys[order], (vals[order] if vals is not None else None), counts

    def local_sort(self, keys, vals, algorithm, lo, hi):
        order = torch.sort(_u(keys), stable=True).indices
        return keys[order], (vals[order] if vals is not None else None)

    def event(self):
        return None

    @staticmethod
    def elapsed(a, b):
        return 0.0


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_total = 20_011
        rng = np.random.default_rng(7)
        if case == "uniform":
            allk = rng.integers(0, 1 << 32, size=n_total, dtype=np.uint64).astype(np.uint32)
        elif case == "small_range":
            allk = rng.integers(0, 5, size=n_total, dtype=np.uint64).astype(np.uint32)
        elif case == "mixture":
            a = rng.integers(0, 1 << 32, size=n_total, dtype=np.uint64)
            b = np.clip(np.rint(2**31 + 2**24 * rng.standard_normal(n_total)), 0, 2**32 - 1).astype(np.uint64)
            allk = np.where(rng.integers(0, 2, size=n_total) > 0, a, b).astype(np.uint32)
        elif case == "sorted":
            allk = np.sort(rng.integers(0, 1 << 32, size=n_total, dtype=np.uint64).astype(np.uint32))
        else:  # one rank empty-ish: all keys equal
            allk = np.full(n_total, 0xFFFFFFFF, dtype=np.uint32)
        # positional shards (uneven on purpose)
        bounds = np.linspace(0, n_total, world + 1).astype(int)
        lo, hi = bounds[rank], bounds[rank + 1]
        keys = torch.from_numpy(allk[lo:hi].view(np.int32).copy())
        vals = torch.arange(lo, hi, dtype=torch.int32)  # global positions: makes stability observable
        sorter = KeyRangeSorter(dist, TorchCpuOps(), sample_per_rank=512)
        k, v, pt = sorter.sort(keys, vals)
        np.save(os.path.join(out_dir, f"k{rank}.npy"), k.numpy().view(np.uint32))
        np.save(os.path.join(out_dir, f"v{rank}.npy"), v.numpy())
        if rank == 0:
            np.save(os.path.join(out_dir, "all.npy"), allk)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", ["uniform", "small_range", "mixture", "sorted", "constant"])
def test_key_range_sort_over_gloo(tmp_path, world, case):
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    allk = np.load(tmp_path / "all.npy")
    ks = [np.load(tmp_path / f"k{r}.npy") for r in range(world)]
    vs = [np.load(tmp_path / f"v{r}.npy") for r in range(world)]
    got_k = np.concatenate(ks)
    got_v = np.concatenate(vs)
    order = np.argsort(allk, kind="stable")
    assert np.array_equal(got_k, allk[order])  # globally sorted, nothing lost
    assert np.array_equal(got_v, order.astype(np.int32))  # stable across ranks
    # ranges are disjoint and ordered
    for a, b in zip(ks, ks[1:]):
        if a.size and b.size:
            assert a[-1] <= b[0]


def test_splitters_balance_uniform(tmp_path):
    """With uniform keys the sampled splitters give near-even ranges."""
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), "uniform", str(tmp_path)), nprocs=world, join=True)
    sizes = [np.load(tmp_path / f"k{r}.npy").size for r in range(world)]
    assert max(sizes) / (sum(sizes) / world) < 1.15


def test_fused_exchange_addresses():
    """Slots of the fused exchange: destination d receives the runs of sources
    0..G-1 back to back, in source order (= global input order)."""
    from paper_1206_3511_b200.partition import fused_destinations, recv_totals

    m = [[3, 0, 5], [1, 2, 0], [4, 4, 4]]  # row = source, column = destination
    assert recv_totals(m) == [8, 6, 9]
    bases = [1000, 2000, 3000]
    assert fused_destinations(m, 0, bases, 4) == [1000, 2000, 3000]
    assert fused_destinations(m, 1, bases, 4) == [1000 + 12, 2000, 3000 + 20]
    assert fused_destinations(m, 2, bases, 4) == [1000 + 16, 2000 + 8, 3000 + 20]
    for d in range(3):  # the last source's run ends exactly at the destination's total
        last = fused_destinations(m, 2, bases, 4)[d] + 4 * m[2][d]
        assert last == bases[d] + 4 * recv_totals(m)[d]


def _fused_fallback_worker(rank, world, port, out_dir):
    """enable_fused on a box where CUDA IPC is unavailable: every rank must take
    the same branch (agreement all-reduce) and keep the NCCL path -- no hang, no
    half-enabled state."""
    from paper_1206_3511_b200 import partition

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sorter = KeyRangeSorter(dist, TorchCpuOps())
        keys = torch.arange(1000, dtype=torch.int32)
        ok = partition.enable_fused(sorter, keys, "radix")
        with open(os.path.join(out_dir, f"fb{rank}.txt"), "w") as f:
            f.write(f"{int(ok)} {int(sorter.peers is None)}")
    finally:
        dist.destroy_process_group()


def test_fused_exchange_falls_back_on_every_rank(tmp_path):
    world = 2
    mp.spawn(_fused_fallback_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert (tmp_path / f"fb{r}.txt").read_text() == "0 1"
