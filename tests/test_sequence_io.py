"""ISRT sequence files: the device loader and the host-side
header/writer, pinned against the unmodified reference (oracle/_ref:
sequence_io.cpp) and against files the reference itself wrote
(tests/golden/reference_*.isrt, made by tests/golden/make_golden.py).

CPU tests cover the header parser and the writer; `gpu` tests stream payloads
into device memory and compare keys, errors and messages with the reference's
read_sequence_file (mirrors test_sequence_io.cpp)."""
from __future__ import annotations

import hashlib
import json
import os
import struct

import numpy as np
import pytest

from oracle.binding import RECORD_DTYPE, OracleError, Reference
from paper_1206_3511_b200 import _lib
from paper_1206_3511_b200 import sequence as sq

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def ref():
    if not Reference.available():
        pytest.skip("oracle/_ref (the reference built here) is not present")
    return Reference()


def good_bytes(keys=(1, 2, 3), header=(1, 0, 999, 7)) -> bytes:
    k = np.asarray(keys, dtype="<u8")
    return b"ISRT\x01" + struct.pack("<4Q", header[0], k.size, header[2], header[3]) + k.tobytes()


def records(keys):
    r = np.empty(len(keys), dtype=RECORD_DTYPE)
    r["key"] = np.asarray(keys, dtype=np.uint64)
    r["tag"] = np.arange(len(keys), dtype=np.uint64)
    return r


def ref_outcome(ref, path):
    try:
        return ("ok", ref.read_sequence_file(str(path))[0])
    except OracleError as e:
        return ("error", str(e))


# ---------------------------------------------------------------- CPU
def test_golden_files_written_by_the_reference_parse():
    with open(os.path.join(GOLDEN, "reference_sequences.json")) as f:
        meta = json.load(f)
    for name, m in meta.items():
        h = sq.read_header(os.path.join(GOLDEN, name))
        assert (h.case_id, h.n, h.range_bound, h.seed) == (m["case_id"], m["n"], m["range_bound"], m["seed"])
        raw = open(os.path.join(GOLDEN, name), "rb").read()[sq.HEADER_BYTES:]
        assert hashlib.sha256(raw).hexdigest() == m["keys_sha256"]


@pytest.mark.parametrize("keys", [[], [5, 3, 3, 900, 0], [0, (1 << 64) - 1, 1 << 40, 7]])
def test_writer_is_byte_identical_to_the_reference(ref, tmp_path, keys):
    ours, theirs = tmp_path / "ours.isrt", tmp_path / "ref.isrt"
    sq.write_sequence(ours, sq.SequenceHeader(2, 0, 0x0102, 1), keys)
    ref.write_sequence_file(str(theirs), (2, 12345, 0x0102, 1), records(keys))  # n comes from the records
    assert ours.read_bytes() == theirs.read_bytes()


def corrupt_cases():
    good = good_bytes()
    return {
        "good": good,
        "bad magic": b"X" + good[1:],
        "bad version": good[:4] + b"\x02" + good[5:],
        "version 0": good[:4] + b"\x00" + good[5:],
        "truncated preamble": good[:3],
        "truncated header": good[:20],
        "empty": b"",
        "header only, n=0": good_bytes(keys=()),
    }


@pytest.mark.parametrize("case", list(corrupt_cases()))
def test_header_errors_match_the_reference(ref, tmp_path, case):
    path = tmp_path / "f.isrt"
    path.write_bytes(corrupt_cases()[case])
    kind, val = ref_outcome(ref, path)
    if kind == "ok":
        h = sq.read_header(path)
        assert (h.case_id, h.n, h.range_bound, h.seed) == val
    else:
        with pytest.raises(sq.SequenceIoError) as e:
            sq.read_header(path)
        assert str(e.value) == val


def test_missing_file(ref):
    with pytest.raises(sq.SequenceIoError, match="cannot open /nonexistent/intsort.isrt for reading"):
        sq.read_header("/nonexistent/intsort.isrt")
    assert ref_outcome(ref, "/nonexistent/intsort.isrt")[1] == "cannot open /nonexistent/intsort.isrt for reading"


def test_loader_validates_arguments_without_device():
    lib = _lib.load()
    h = _lib.SequenceHeaderC()
    assert lib.isort_sequence_load(b"/nonexistent", None, 0, 3, h, 0) == _lib.ISORT_EINVAL


# ---------------------------------------------------------------- GPU
def dev_load(path, key_bytes):
    hdr, keys = sq.load(path, key_bytes=key_bytes)
    host = keys.cpu().numpy().view(np.uint32 if key_bytes == 4 else np.uint64)
    return hdr, host


@pytest.mark.gpu
def test_device_load_matches_reference_reader(cuda, ref):
    for name in ("reference_case6.isrt", "reference_case1_2p40.isrt"):
        path = os.path.join(GOLDEN, name)
        want_hdr, want = ref.read_sequence_file(path)
        hdr, got = dev_load(path, 8)
        assert (hdr.case_id, hdr.n, hdr.range_bound, hdr.seed) == want_hdr
        assert np.array_equal(got, want["key"])
        _, rec = sq.read_sequence(path)  # the read_sequence_file mirror: tag = position
        assert (rec == want).all()
    hdr, got32 = dev_load(os.path.join(GOLDEN, "reference_case6.isrt"), 4)  # keys < 2^32
    assert np.array_equal(got32.astype(np.uint64), ref.read_sequence_file(
        os.path.join(GOLDEN, "reference_case6.isrt"))[1]["key"])


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 65_535, 65_536, 4 * (1 << 20) + 3, 9_000_001])
def test_device_load_across_staging_chunks_then_sort(cuda, oracle, tmp_path, n):
    import torch

    from paper_1206_3511_b200 import device

    rng = np.random.default_rng(n)
    keys = rng.integers(0, 1 << 32, size=n, dtype=np.uint64)
    path = tmp_path / "u32.isrt"
    sq.write_sequence(path, sq.SequenceHeader(1, 0, (1 << 32) - 1, 42), keys)
    hdr, dkeys = sq.load(path, key_bytes=4)
    assert hdr.n == n
    assert np.array_equal(dkeys.cpu().numpy().view(np.uint32), keys.astype(np.uint32))
    if n:
        s = device.Sorter(n, 4, "bucket", "iota", range_bound=hdr.range_bound)
        k, v = s(dkeys)
        torch.cuda.synchronize()
        want_k, want_i = oracle.sort_u32(keys.astype(np.uint32), with_index=True)
        assert np.array_equal(k.cpu().numpy().view(np.uint32), want_k)
        assert np.array_equal(v.cpu().numpy().view(np.uint32), want_i)


@pytest.mark.gpu
def test_device_load_errors_match_reference(cuda, ref, tmp_path):
    """key > M named by value and position; truncation; and their order, which
    follows the reference's 65,536-key chunked read (sequence_io.cpp:100-117)."""
    n = 300_000
    rng = np.random.default_rng(5)
    base = rng.integers(0, 1000, size=n, dtype=np.uint64)
    cases = {}
    for pos in (0, 65_535, 65_536, 250_001, n - 1):
        k = base.copy()
        k[pos] = 1000 + pos
        k[min(pos + 7, n - 1)] = 5000  # a later bad key must not be the one reported
        cases[f"bad@{pos}"] = (k, None)
    cases["truncated"] = (base, 3)
    bad_early = base.copy()
    bad_early[1000] = 77777
    cases["bad in a complete chunk, then truncated"] = (bad_early, 8 * 1000 + 5)
    bad_late = base.copy()
    bad_late[n - 10] = 77777
    cases["bad in the short chunk"] = (bad_late, 8 * 20)
    for name, (k, cut) in cases.items():
        path = tmp_path / "e.isrt"
        sq.write_sequence(path, sq.SequenceHeader(1, 0, 999, 7), k)
        if cut:
            data = path.read_bytes()
            path.write_bytes(data[: len(data) - cut])
        kind, msg = ref_outcome(ref, path)
        assert kind == "error", name
        for kb in (4, 8):
            with pytest.raises(sq.SequenceIoError) as e:
                sq.load(path, key_bytes=kb)
            assert str(e.value) == msg, (name, kb)


@pytest.mark.gpu
def test_u32_load_rejects_wide_keys(cuda, tmp_path):
    path = tmp_path / "w.isrt"
    sq.write_sequence(path, sq.SequenceHeader(1, 0, 1 << 40, 1), [1, 2, (1 << 32) + 5, 3])
    with pytest.raises(_lib.IsortError, match="position 2 does not fit 32 bits"):
        sq.load(path, key_bytes=4)
    hdr, got = dev_load(path, 8)
    assert got.tolist() == [1, 2, (1 << 32) + 5, 3]
