"""Minimal driver for ncu captures: sort `n` seeded keys `reps` times with one algorithm.

    python tools/prof_sort.py --alg radix --n 100000000 --reps 2 [--vals iota] [--config c2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_1206_3511_b200 import device, inputs

p = argparse.ArgumentParser()
p.add_argument("--alg", default="radix")
p.add_argument("--n", type=int, default=100_000_000)
p.add_argument("--reps", type=int, default=2)
p.add_argument("--vals", default=None)
p.add_argument("--config", default="c2")
a = p.parse_args()
keys = inputs.config_keys(a.config, a.n)
t = torch.from_numpy(keys.view(np.int32)).cuda()
s = device.Sorter(a.n, 4, a.alg, a.vals, range_bound=inputs.config_range_bound(a.config))
for _ in range(a.reps):
    s(t)
torch.cuda.synchronize()
out = s.keys_out.cpu().numpy().view(np.uint32)
assert np.all(out[:-1] <= out[1:]), "unsorted"
print("ok", a.alg, a.n)
