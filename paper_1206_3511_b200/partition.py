"""Multi-GPU sort by key-range partitioning.

The reference is single-threaded and lists parallel sorting as future work
(SPEC.md:8); this is the engine's scale-out step.  One process
per GPU (torch.distributed, NCCL over NVLink/NVSwitch); rank r starts with the
r-th positional shard of the input and ends with the r-th key range of the
sorted output, so the global result is the rank-ordered concatenation:

  1. sample      every rank takes S evenly spaced keys of its shard (device)
  2. splitters   all_gather of the samples, device radix sort, the G-1 quantiles
                 (key values: equal keys never straddle two ranks)
  3. partition   one stable one-sweep pass with a destination-rank digitizer
                 (isort_partition_u32): the shard grouped by destination, input
                 order kept inside each group; per-destination counts
  4. counts      all_gather of the G x G count matrix
  5. exchange    all_to_all_single (NCCL grouped send/recv): chunks land ordered
                 by source rank, i.e. in global input order
  6. local sort  stable radix or bucket sort of the received keys

Stability: received chunks are in source-rank (= input) order and the local
sort is stable, so keys with equal value keep their global input order, and
the concatenation over ranks equals the single-device stable sort bit for bit.

Step 3 and 6 are CUDA kernels (via :class:`CudaOps`); steps 1-2 and 4-5 are
collectives.

Fused exchange (:class:`PeerBuffers`, SURVEY 8e "fused variant"): every rank's
receive buffer is mapped into every process (CUDA IPC over NVLink/NVSwitch).
Step 3 is split into a count (the destination-digit histogram) and the
partition pass itself; after the G x G count matrix is gathered, the partition
kernel stores each destination's run straight into its slot in that rank's
receive buffer (isort_partition_scatter_u32), so steps 3 and 5 are one kernel
and the send buffer disappears.  An on-stream all-reduce orders the local sort
after every peer's stores.  The first distributed sort checks the fused result
against the NCCL path bit for bit; any error or mismatch falls back to NCCL.  The protocol itself (:class:`KeyRangeSorter`) only talks to an
ops object, which lets tests drive it over gloo on CPU with a torch-CPU stand-in
for the kernels (tests/test_partition_gloo.py); the product path always uses
CudaOps.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import torch

from . import _lib

DEFAULT_SAMPLE = 1 << 16


@dataclass
class PhaseTimes:
    """Per-phase device times (ms) of one distributed sort on this rank."""

    splitters: float = 0.0
    partition: float = 0.0
    exchange: float = 0.0
    local_sort: float = 0.0
    received: int = 0
    extra: dict = field(default_factory=dict)
    events: tuple = ()

    def resolve(self, ops) -> "PhaseTimes":
        """Turn the recorded events into per-phase times (waits for the last one)."""
        if self.events:
            e0, e1, e2, e3, e4 = self.events
            self.splitters = ops.elapsed(e0, e1)
            self.partition = ops.elapsed(e1, e2)
            self.exchange = ops.elapsed(e2, e3)
            self.local_sort = ops.elapsed(e3, e4)
            self.events = ()
        return self


class CudaOps:
    """Kernels of the distributed sort on this rank's GPU (libisort.so)."""

    def __init__(self, device: torch.device):
        self.device = device
        self.lib = _lib.load()

    def sample(self, keys: torch.Tensor, s: int) -> torch.Tensor:
        """Exactly s keys: evenly spaced positions (cyclic when n < s); an empty
        shard contributes the largest key value (it only shifts quantiles)."""
        n = keys.numel()
        if n == 0:
            return torch.full((s,), -1, dtype=keys.dtype, device=keys.device)
        pos = (torch.arange(s, device=keys.device, dtype=torch.int64) * n) // s
        return keys[pos].contiguous()

    def sort(self, keys: torch.Tensor) -> torch.Tensor:
        from .device import radix_sort

        k, _ = radix_sort(keys)
        return k

    def partition(self, keys, vals, splitters: list[int], parts: int):
        n = keys.numel()
        vmode = _lib.VALS_LOAD if vals is not None else _lib.VALS_NONE
        out = torch.empty_like(keys)
        vout = torch.empty_like(vals) if vals is not None else None
        counts = torch.zeros(parts, dtype=torch.int64, device=self.device)
        tb = self.lib.isort_partition_temp_bytes(n, 4, vmode)
        temp = torch.empty(max(tb, 1), dtype=torch.uint8, device=self.device)
        import ctypes

        spl = (ctypes.c_uint32 * max(1, parts - 1))(*[int(x) & 0xFFFFFFFF for x in splitters])
        s = torch.cuda.current_stream(self.device).cuda_stream
        _lib.check(self.lib.isort_partition_u32(keys.data_ptr(), out.data_ptr(),
                                                vals.data_ptr() if vals is not None else None,
                                                vout.data_ptr() if vout is not None else None,
                                                n, spl, parts, vmode, counts.data_ptr(), temp.data_ptr(), tb, s))
        return out, vout, counts

    def _temp(self, n: int):
        tb = self.lib.isort_partition_temp_bytes(n, 4, _lib.VALS_LOAD)
        if getattr(self, "_tbuf", None) is None or self._tbuf.numel() < tb:
            self._tbuf = torch.empty(max(tb, 1), dtype=torch.uint8, device=self.device)
        return self._tbuf, tb

    def partition_counts(self, keys, splitters: list[int], parts: int):
        """Fused path, step 1: per-destination counts (state kept for step 2)."""
        import ctypes

        n = keys.numel()
        temp, tb = self._temp(n)
        counts = torch.zeros(parts, dtype=torch.int64, device=self.device)
        spl = (ctypes.c_uint32 * max(1, parts - 1))(*[int(x) & 0xFFFFFFFF for x in splitters])
        s = torch.cuda.current_stream(self.device).cuda_stream
        _lib.check(self.lib.isort_partition_counts_u32(keys.data_ptr(), n, spl, parts, counts.data_ptr(),
                                                       temp.data_ptr(), tb, s))
        return counts

    def partition_scatter_table(self, keys, vals, splitters: list[int], parts: int, table: torch.Tensor):
        """Fused path, step 2 with the destination table on the device (int64,
        [key bases..., payload bases...]): no host read of the count matrix."""
        import ctypes

        n = keys.numel()
        temp, tb = self._temp(n)
        spl = (ctypes.c_uint32 * max(1, parts - 1))(*[int(x) & 0xFFFFFFFF for x in splitters])
        vmode = _lib.VALS_LOAD if vals is not None else _lib.VALS_NONE
        s = torch.cuda.current_stream(self.device).cuda_stream
        _lib.check(self.lib.isort_partition_scatter_table_u32(
            keys.data_ptr(), vals.data_ptr() if vals is not None else None, n, spl, parts, vmode, table.data_ptr(),
            temp.data_ptr(), tb, s))

    def partition_scatter(self, keys, vals, splitters: list[int], parts: int, key_dst: list[int],
                          val_dst: list[int] | None):
        """Fused path, step 2: the partition pass storing each destination's run at key_dst[d]."""
        import ctypes

        n = keys.numel()
        temp, tb = self._temp(n)
        spl = (ctypes.c_uint32 * max(1, parts - 1))(*[int(x) & 0xFFFFFFFF for x in splitters])
        kd = (ctypes.c_void_p * parts)(*key_dst)
        vd = (ctypes.c_void_p * parts)(*(val_dst or [0] * parts))
        vmode = _lib.VALS_LOAD if vals is not None else _lib.VALS_NONE
        s = torch.cuda.current_stream(self.device).cuda_stream
        _lib.check(self.lib.isort_partition_scatter_u32(keys.data_ptr(), vals.data_ptr() if vals is not None else None,
                                                        n, spl, parts, vmode, kd, vd if vals is not None else None,
                                                        temp.data_ptr(), tb, s))

    def local_sort(self, keys, vals, algorithm: str, lo: int, hi: int):
        from . import device

        if keys.numel() == 0:
            return keys, vals
        if algorithm == "bucket":
            # n buckets over this rank's key range [lo, hi], not [0, hi]: a rank
            # high in the key space (or a narrow, dense range) keeps ~1 key per bucket
            k, v = device.bucket_sort(keys, hi, vals=vals, range_lo=lo)
        else:
            k, v = device.radix_sort(keys, vals=vals)
        return k, v

    def event(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    @staticmethod
    def elapsed(a, b) -> float:
        b.synchronize()
        return a.elapsed_time(b)


def _all_to_all(dist, out, inp, recv, send):
    """all_to_all_single (NCCL over NVLink); under gloo (plumbing checks, CPU
    tests) CUDA tensors are staged through host memory."""
    if out.is_cuda and dist.get_backend() == "gloo":
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(o, inp.cpu(), output_split_sizes=recv, input_split_sizes=send)
        out.copy_(o)
    else:
        dist.all_to_all_single(out, inp, output_split_sizes=recv, input_split_sizes=send)


def recv_totals(matrix: list[list[int]]) -> list[int]:
    """Keys each rank receives: column sums of the count matrix (row = source)."""
    g = len(matrix)
    return [sum(matrix[src][d] for src in range(g)) for d in range(g)]


def fused_destinations(matrix: list[list[int]], me: int, bases: list[int], elem_bytes: int) -> list[int]:
    """Device address where rank `me`'s run for destination d starts: d's receive
    buffer + the keys of lower source ranks (chunks land in source-rank order)."""
    g = len(matrix)
    return [bases[d] + elem_bytes * sum(matrix[src][d] for src in range(me)) for d in range(g)]


class _CudaArray:
    """A raw device pointer seen as a tensor (torch.as_tensor via __cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (ptr, False), "version": 3,
                                         "strides": None}


def device_view(ptr: int, n: int, device) -> torch.Tensor:
    if n == 0:
        return torch.empty(0, dtype=torch.int32, device=device)
    return torch.as_tensor(_CudaArray(ptr, n), device=device)


class PeerBuffers:
    """Receive buffers (keys + u32 payload) of all ranks, mapped into this process.

    Each rank allocates `capacity` keys with isort_ipc_alloc, the 64-byte IPC
    handles are all-gathered, and every peer's buffers are opened with
    isort_ipc_open (peer access over NVLink).  `key_bases[r]` / `val_bases[r]`
    are device addresses usable by this rank's kernels."""

    def __init__(self, dist, device: torch.device, capacity: int):
        import ctypes

        self.lib = _lib.load()
        self.dist, self.device, self.capacity = dist, device, capacity
        g, me = dist.get_world_size(), dist.get_rank()
        dev_index = device.index if device.index is not None else 0
        self.own, self.opened, handles = [], [], []
        ok = torch.ones(1, dtype=torch.int32, device=device)
        try:
            for _ in range(2):  # keys, payload
                ptr = ctypes.c_void_p()
                h = (ctypes.c_ubyte * 64)()
                _lib.check(self.lib.isort_ipc_alloc(4 * max(capacity, 1), dev_index, ctypes.byref(ptr), h))
                self.own.append(int(ptr.value))
                handles.append(bytes(h))
        except Exception:  # noqa: BLE001 - any local failure: every rank must still reach _agree
            ok.zero_()
            handles = [bytes(64), bytes(64)]
        self._agree(ok, "allocate")  # every rank takes the same branch before the next collective
        mine = torch.tensor(list(handles[0] + handles[1]), dtype=torch.uint8, device=device)
        allh = [torch.zeros_like(mine) for _ in range(g)]
        dist.all_gather(allh, mine)
        self.key_bases, self.val_bases = [], []
        try:
            for r in range(g):
                if r == me:
                    self.key_bases.append(self.own[0])
                    self.val_bases.append(self.own[1])
                    continue
                raw = bytes(allh[r].cpu().tolist())
                ptrs = []
                for i in range(2):
                    ptr = ctypes.c_void_p()
                    hb = (ctypes.c_ubyte * 64).from_buffer_copy(raw[64 * i: 64 * (i + 1)])
                    _lib.check(self.lib.isort_ipc_open(hb, dev_index, ctypes.byref(ptr)))
                    self.opened.append(int(ptr.value))
                    ptrs.append(int(ptr.value))
                self.key_bases.append(ptrs[0])
                self.val_bases.append(ptrs[1])
        except Exception:  # noqa: BLE001
            ok.zero_()
        self._agree(ok, "open")
        self.key_table = torch.tensor(self.key_bases, dtype=torch.int64, device=device)
        self.val_table = torch.tensor(self.val_bases, dtype=torch.int64, device=device)

    def _agree(self, ok: torch.Tensor, what: str) -> None:
        self.dist.all_reduce(ok, op=self.dist.ReduceOp.MIN)
        if not bool(ok.item()):
            self.close()
            raise RuntimeError(f"PeerBuffers: some rank could not {what} its CUDA IPC buffers")

    def close(self):
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)
        if self.dist.get_world_size() > 1:
            self.dist.barrier()  # no peer still writes into our buffers
        for p in self.opened:
            self.lib.isort_ipc_close(p)
        for p in self.own:
            self.lib.isort_ipc_free(p)
        self.opened, self.own = [], []


class KeyRangeSorter:
    """Distributed stable sort of u32 keys (+ optional u32 payload) over a process group."""

    def __init__(self, dist, ops, sample_per_rank: int = DEFAULT_SAMPLE, key_max: int = 0xFFFFFFFF,
                 peers: PeerBuffers | None = None):
        self.dist = dist
        self.ops = ops
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self.sample_per_rank = sample_per_rank
        self.key_max = key_max
        self.peers = peers  # fused partition + exchange when set
        self.last_path = None

    def splitters(self, keys: torch.Tensor) -> list[int]:
        """G-1 ascending splitter key values from the gathered sample's quantiles.

        Every rank contributes exactly `sample_per_rank` keys (a strided sample,
        repeated cyclically when the shard is smaller; an empty shard sends the
        largest key), so one all_gather of fixed size suffices and the only host
        read is the G-1 splitters themselves -- kernel parameters of the
        partition pass (DestDigitizer): compared in registers against constant-bank
        operands, cheaper per key than any device-memory lookup."""
        g = self.world
        if g == 1:
            return []
        smp = self.ops.sample(keys, self.sample_per_rank)
        gathered = [torch.empty_like(smp) for _ in range(g)]
        self.dist.all_gather(gathered, smp)
        srt = self.ops.sort(torch.cat(gathered))
        # quantile i*len/g (as unsigned key values); equal keys never straddle ranks
        m = srt.numel()
        idx = torch.tensor([min(m - 1, (i * m) // g) for i in range(1, g)], device=srt.device)
        out = [int(v) & 0xFFFFFFFF for v in srt[idx].tolist()]
        for i in range(1, len(out)):  # ascending (duplicates allowed: empty ranges)
            out[i] = max(out[i], out[i - 1])
        return out

    def _fused_exchange(self, keys, vals, spl):
        """Counts -> gathered count matrix -> partition pass storing into the peers'
        receive buffers -> on-stream barrier.  Returns (keys, payload) views of this
        rank's receive buffer, or None when some rank's share exceeds the capacity.

        The count matrix stays on the device: the destination table (peer base +
        the runs of lower source ranks, fused_destinations) is computed there and
        the partition kernel reads it from device memory.  The host reads only this
        rank's received total and the largest total (the local sort's size and the
        capacity check), with the copy queued behind the partition kernel so the
        round trip overlaps it."""
        g, me, pb = self.world, self.rank, self.peers
        counts = self.ops.partition_counts(keys, spl, g)
        allc = [torch.zeros_like(counts) for _ in range(g)]
        self.dist.all_gather(allc, counts)
        matrix = torch.stack(allc)  # row = source rank, column = destination rank (int64, device)
        totals = matrix.sum(dim=0)
        before = matrix[:me].sum(dim=0) if me > 0 else torch.zeros_like(totals)  # runs of lower source ranks
        fits = totals.max() <= pb.capacity
        table = torch.cat([pb.key_table + 4 * before, pb.val_table + 4 * before])
        table = torch.where(fits, table, torch.zeros_like(table))  # never store out of bounds
        self.ops.partition_scatter_table(keys, vals, spl, g, table)
        info = torch.stack([totals[me], fits.to(totals.dtype)]).cpu()  # after the kernel in stream order
        if not bool(info[1]):
            return None
        total = int(info[0])
        flag = torch.zeros(1, dtype=torch.int32, device=keys.device)
        self.dist.all_reduce(flag)  # every peer's stores precede the local sort
        out = device_view(pb.key_bases[me], total, keys.device)
        vout = device_view(pb.val_bases[me], total, keys.device) if vals is not None else None
        return out, vout

    def sort(self, keys: torch.Tensor, vals: torch.Tensor | None = None, algorithm: str = "radix",
             force_nccl: bool = False, resolve: bool = True):
        """Returns (this rank's sorted key range, payload or None, PhaseTimes).
        resolve=False leaves the phase events unread (PhaseTimes.resolve later), so
        back-to-back sorts are not serialised by the timing."""
        g, me = self.world, self.rank
        pt = PhaseTimes()
        e0 = self.ops.event()
        spl = self.splitters(keys)
        e1 = self.ops.event()
        fused = None
        if g > 1 and self.peers is not None and not force_nccl:
            fused = self._fused_exchange(keys, vals, spl)  # None: does not fit, use NCCL
        if g > 1 and fused is None:
            parted, pvals, counts = self.ops.partition(keys, vals, spl, g)
            self.last_path = "nccl"
        elif g > 1:
            parted, pvals, counts = None, None, None
            self.last_path = "fused"
        else:
            parted, pvals, counts = keys, vals, None
        e2 = self.ops.event()
        if g > 1 and fused is not None:
            out, vout = fused
        elif g > 1:
            # count matrix: row = source rank, column = destination rank
            allc = [torch.zeros_like(counts) for _ in range(g)]
            self.dist.all_gather(allc, counts)
            # all_to_all_single takes its split sizes on the host: one read of both
            sr = torch.cat([counts, torch.stack(allc)[:, me]]).tolist()
            send, recv = [int(x) for x in sr[:g]], [int(x) for x in sr[g:]]
            out = torch.empty(sum(recv), dtype=keys.dtype, device=keys.device)
            _all_to_all(self.dist, out, parted, recv, send)
            vout = None
            if vals is not None:
                vout = torch.empty(sum(recv), dtype=vals.dtype, device=vals.device)
                _all_to_all(self.dist, vout, pvals, recv, send)
        else:
            out, vout = parted, pvals
        e3 = self.ops.event()
        lo = spl[me - 1] if me > 0 else 0
        hi = (spl[me] - 1) if me < g - 1 and spl[me] > 0 else self.key_max
        hi = max(hi, lo)
        sk, sv = self.ops.local_sort(out, vout, algorithm, lo, hi)
        e4 = self.ops.event()
        pt.events = (e0, e1, e2, e3, e4)
        if resolve:
            pt.resolve(self.ops)
        pt.received = int(out.numel())
        return sk, sv, pt


def enable_fused(sorter: KeyRangeSorter, keys: torch.Tensor, algorithm: str, slack: float = 1.5) -> bool:
    """Map the receive buffers (capacity = slack x the local shard) and switch the
    sorter to the fused exchange if one trial sort matches the NCCL path bit for
    bit on every rank; otherwise (IPC unavailable, mismatch) keep NCCL."""
    dist, dev = sorter.dist, keys.device
    try:
        sorter.peers = PeerBuffers(dist, dev, int(slack * keys.numel()) + (1 << 16))
    except RuntimeError:  # raised on every rank alike
        sorter.peers = None
        return False
    ok = torch.ones(1, dtype=torch.int32, device=dev)
    pos = torch.arange(keys.numel(), dtype=torch.int32, device=dev)
    a_k, a_v, _ = sorter.sort(keys, pos, algorithm=algorithm)
    path = sorter.last_path
    a_k, a_v = a_k.clone(), a_v.clone()
    b_k, b_v, _ = sorter.sort(keys, pos, algorithm=algorithm, force_nccl=True)
    if path != "fused" or not (torch.equal(a_k, b_k) and torch.equal(a_v, b_v)):
        ok.zero_()
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if not bool(ok.item()):
        sorter.peers.close()
        sorter.peers = None
    return sorter.peers is not None


def bench_distributed(keys: torch.Tensor, algorithm: str, range_bound: int, steps: int, warmup: int, dist):
    """Time `steps` distributed sorts of the per-rank shards (bench.py, N > 1).

    Device time per step = max over ranks of (CUDA-event time from the barrier
    to the end of the last local sort) / steps.  Returns (ms_per_step, info,
    this rank's sorted key range from the last step)."""
    import os

    dev = keys.device
    ops = CudaOps(dev)
    sorter = KeyRangeSorter(dist, ops)
    try:
        if os.environ.get("ISORT_FUSED_EXCHANGE", "1") != "0":
            enable_fused(sorter, keys, algorithm)
        l0 = _lib.load().isort_launch_count()
        for _ in range(warmup):
            sorter.sort(keys, algorithm=algorithm)
        torch.cuda.synchronize(dev)
        dist.barrier()
        torch.cuda.synchronize(dev)
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        phases = []
        l1 = _lib.load().isort_launch_count()
        start.record()
        for _ in range(steps):
            sk, _, pt = sorter.sort(keys, algorithm=algorithm, resolve=False)
            phases.append(pt)
        end.record()
        torch.cuda.synchronize(dev)
        launches = _lib.load().isort_launch_count() - l1
        for p in phases:
            p.resolve(ops)
        ms = torch.tensor([start.elapsed_time(end) / steps], device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        avg = {k: sum(getattr(p, k) for p in phases) / len(phases)
               for k in ("splitters", "partition", "exchange", "local_sort")}
        recv = torch.tensor([float(phases[-1].received)], device=dev)
        mx = recv.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        mean = recv.clone()
        dist.all_reduce(mean, op=dist.ReduceOp.SUM)
        info = {"phases_ms": {k: round(v, 4) for k, v in avg.items()}, "launches": int(launches),
                "max_over_mean_received": float(mx.item() / max(1.0, mean.item() / dist.get_world_size())),
                "warmup_launches": int(l1 - l0),
                "exchange": "fused (partition stores into peer receive buffers over NVLink)"
                if sorter.peers is not None else "nccl all_to_all"}
        return float(ms.item()), info, sk.clone()
    finally:
        if sorter.peers is not None:
            sorter.peers.close()
            sorter.peers = None


def _wallclock() -> float:  # pragma: no cover - helper for ad-hoc use
    return time.perf_counter()
