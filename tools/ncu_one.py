"""One sort of a 1e8-key case (for an ncu launch list): python tools/ncu_one.py KIND ALG VALS
KIND as in tools/time_sorts.py; VALS none|iota."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1206_3511_b200 import device  # noqa: E402
from tools.time_sorts import keys_for  # noqa: E402

kind, alg, vals = sys.argv[1], sys.argv[2], sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 100_000_000
k = keys_for(n, kind)
t = torch.from_numpy(k.view(np.int32)).cuda()
bound = int(kind.split(":")[1]) if kind.startswith("below:") else (1 << 32) - 1
s = device.Sorter(n, 4, alg, None if vals == "none" else vals, range_bound=bound)
for _ in range(2):
    s(t)
torch.cuda.synchronize()
print("ok")
