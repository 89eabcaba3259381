"""CPU checks of the full-size parity fixtures (tests/golden/full_size_checksums.json):
every BASELINE configuration has an entry, and the harness input builders
reproduce the checksummed inputs (C2 and C3 here; C4a/C4b/C5 are checked by the
GPU test that rebuilds them)."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).astype("<u4", copy=False).tobytes()).hexdigest()


def test_every_config_has_a_reference_checksum():
    with open(os.path.join(GOLDEN, "full_size_checksums.json")) as f:
        c = json.load(f)
    assert set(c) == {"c1", "c2", "c3", "c4a", "c4b", "c5"}
    assert c["c5"]["n"] == 10**9 and c["c1"]["n"] == 10**6 and all(c[k]["n"] == 10**8 for k in ("c2", "c3", "c4a", "c4b"))
    assert "reference radix_sort_lsd" in c["c2"]["source"]


def test_input_builders_match_checksummed_inputs():
    from paper_1206_3511_b200 import inputs

    with open(os.path.join(GOLDEN, "full_size_checksums.json")) as f:
        c = json.load(f)
    for cfg in ("c2", "c3"):
        assert sha(inputs.config_keys(cfg)) == c[cfg]["input_sha256"], cfg
