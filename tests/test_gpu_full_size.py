"""Bit-exact parity at BASELINE.json's stated sizes, for every configuration.

tests/golden/full_size_checksums.json holds SHA-256 digests of the reference's
own output (tests/golden/make_full_size.py):
  * C2, C3, C4a (10^8 keys from the reference's generate()) and C4b (C4a
    reversed, tags = positions): the UNMODIFIED reference radix_sort_lsd at base
    256 (proj/core/src/sort.cpp:112-119), cross-checked equal to its
    bucket_sort (sort.cpp:136-152);
  * C5 (10^9-key mixture, a harness addition): the oracle's keys + stable
    positions restatement of the same LSD sort.
Each GPU sort (radix and bucket, with and without the position payload) must
reproduce the sorted keys AND the stable positions (the records' tags) bit for
bit.  Inputs are rebuilt here and their digest checked first, so a generator
difference cannot pass as a sort difference.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).astype("<u4", copy=False).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def checks():
    with open(os.path.join(GOLDEN, "full_size_checksums.json")) as f:
        return json.load(f)


def config_input(cfg: str, oracle) -> np.ndarray:
    from paper_1206_3511_b200 import inputs

    if cfg == "c5":  # Box-Muller through the oracle's libm, as the checksum was made
        return oracle.mixture_u32(10**9, 42)
    return inputs.config_keys(cfg)


def sort_on_device(keys: np.ndarray, algorithm: str, payload, bound: int):
    import torch

    from paper_1206_3511_b200 import device

    t = torch.from_numpy(keys.view(np.int32)).cuda()
    s = device.Sorter(keys.size, 4, algorithm, payload, range_bound=bound)
    k, v = s(t)
    torch.cuda.synchronize()
    ko = k.cpu().numpy().view(np.uint32)
    vo = v.cpu().numpy().view(np.uint32) if v is not None else None
    del s, t, k, v
    torch.cuda.empty_cache()
    return ko, vo


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4a", "c4b", "c5"])
def test_full_size_bit_exact(cuda, oracle, checks, cfg):
    c = checks[cfg]
    keys = config_input(cfg, oracle)
    assert keys.size == c["n"]
    assert sha(keys) == c["input_sha256"], f"{cfg}: input generator differs from the checksummed input"
    bound = int(c["range_bound"])
    for alg in ("radix", "bucket"):
        ko, vo = sort_on_device(keys, alg, "iota", bound)
        assert sha(ko) == c["sorted_keys_sha256"], f"{cfg} {alg}: sorted keys differ from the reference"
        assert sha(vo) == c["stable_positions_sha256"], f"{cfg} {alg}: stable positions differ from the reference"
        del ko, vo
        ko, _ = sort_on_device(keys, alg, None, bound)
        assert sha(ko) == c["sorted_keys_sha256"], f"{cfg} {alg} (keys only): sorted keys differ"
        del ko


def test_beyond_2_pow_30_keys_per_call(cuda):
    """n > 2^30: the passes switch to 64-bit look-back status words (a 32-bit
    word's 30-bit count would overflow).  A stable sort is unique, so checking
    (a) keys sorted, (b) keys_out == keys_in[positions] (a permutation that carries
    each key) and (c) positions ascending inside every run of equal keys (there are
    ~10^8 such pairs among 2^30 random u32 keys) proves bit-exactness at this size."""
    from paper_1206_3511_b200 import _lib, inputs

    n = (1 << 30) + 12_345
    assert n > 2**30 and n <= _lib.load().isort_max_keys()
    keys = inputs.uniform_u32(n, seed=2026)
    for alg in ("radix", "bucket"):
        ko, vo = sort_on_device(keys, alg, "iota", (1 << 32) - 1)
        assert bool(np.all(ko[1:] >= ko[:-1])), alg
        assert np.array_equal(keys[vo], ko), alg
        eq = ko[1:] == ko[:-1]
        assert int(eq.sum()) > 10**7
        assert bool(np.all(vo[1:][eq] > vo[:-1][eq])), f"{alg}: unstable"
        del ko, vo, eq
