"""W processes (default 2) on ONE GPU running the fused exchange end to end (CUDA IPC
between the processes, gloo for the host-side collectives): checks that the
partition kernel of each rank lands its runs in the other rank's receive buffer
and that the rank-ordered result equals the global stable sort.  No kernel of
one rank waits on a kernel of the other; only the host collectives synchronise.

    python tools/two_rank_fused_check.py [n] [world] [radix|bucket]
"""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def worker(rank, world, port, n, out, algorithm):
    from paper_1206_3511_b200 import inputs, partition

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    keys = inputs.mixture_u32(n, 7)
    sh = np.array_split(np.arange(n), world)[rank]
    k = torch.from_numpy(keys[sh].view(np.int32)).to(dev)
    pos = torch.from_numpy(sh.astype(np.int32)).to(dev)
    sorter = partition.KeyRangeSorter(dist, partition.CudaOps(dev))
    sorter.peers = partition.PeerBuffers(dist, dev, int(1.5 * k.numel()) + (1 << 16))
    sk, sv, pt = sorter.sort(k, pos, algorithm=algorithm)
    torch.cuda.synchronize()
    np.save(os.path.join(out, f"k{rank}.npy"), sk.cpu().numpy().view(np.uint32))
    np.save(os.path.join(out, f"v{rank}.npy"), sv.cpu().numpy())
    with open(os.path.join(out, f"path{rank}.txt"), "w") as f:
        f.write(sorter.last_path or "none")
    sorter.peers.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    import tempfile

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_017
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    algorithm = sys.argv[3] if len(sys.argv) > 3 else "radix"
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tempfile.mkdtemp()
    mp.spawn(worker, args=(world, port, n, out, algorithm), nprocs=world, join=True)
    from paper_1206_3511_b200 import inputs

    keys = inputs.mixture_u32(n, 7)
    order = np.argsort(keys, kind="stable")
    gk = np.concatenate([np.load(os.path.join(out, f"k{r}.npy")) for r in range(world)])
    gv = np.concatenate([np.load(os.path.join(out, f"v{r}.npy")) for r in range(world)])
    paths = [open(os.path.join(out, f"path{r}.txt")).read() for r in range(world)]
    ok = np.array_equal(gk, keys[order]) and np.array_equal(gv.astype(np.int64), order)
    print(f"paths={paths} n={n} algorithm={algorithm} bit-exact={ok}")
    sys.exit(0 if ok and paths == ["fused"] * world else 1)
