import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1206_3511_b200 import device, _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
k = np.random.default_rng(1).integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
t = torch.from_numpy(k.view(np.int32)).cuda()
s = device.Sorter(n, 4, "bucket", None, range_bound=(1 << 32) - 1)
ko, _ = s(t)
torch.cuda.synchronize()
got = ko.cpu().numpy().view(np.uint32)
want = np.sort(k)
bad = np.nonzero(got != want)[0]
print("n", n, "mismatches", bad.size, "first", bad[:5])
