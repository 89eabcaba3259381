"""ISRT sequence files on the device.

Mirror of the reference's sequence_io API (proj/core/include/intsort/sequence_io.hpp,
proj/core/src/sequence_io.cpp) for the sort path's input side:

* ``read_header(path)``     -- header parse + validation (sequence_io.cpp:72-91);
* ``load(path, key_bytes)`` -- the n keys streamed straight into a device tensor,
  range-checked on the device (sequence_io.cpp:93-119), ready for ``device.Sorter``;
* ``read_sequence(path)``   -- the reference's ``read_sequence_file``: header plus a
  record array with tag = position;
* ``write_sequence(path, header, keys)`` -- the writer (sequence_io.cpp:45-70),
  host-side, used to produce inputs.

Errors raise :class:`SequenceIoError` with the reference's messages.
"""
from __future__ import annotations

import ctypes
import os
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import SequenceIoError  # noqa: F401  (re-export)

MAGIC = b"ISRT"
VERSION = 1
HEADER_BYTES = 5 + 4 * 8


@dataclass
class SequenceHeader:
    case_id: int = 0
    n: int = 0
    range_bound: int = 0
    seed: int = 0


def _hdr(c: _lib.SequenceHeaderC) -> SequenceHeader:
    return SequenceHeader(int(c.case_id), int(c.n), int(c.range_bound), int(c.seed))


def write_sequence(path: str | os.PathLike, header: SequenceHeader, keys) -> None:
    """write_sequence_file (sequence_io.cpp:45-70): header.n is taken from len(keys)."""
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))
    with open(path, "wb") as f:
        f.write(MAGIC + bytes([VERSION]))
        f.write(struct.pack("<4Q", header.case_id, k.size, header.range_bound, header.seed))
        f.write(k.astype("<u8").tobytes())


def read_header(path: str | os.PathLike) -> SequenceHeader:
    h = _lib.SequenceHeaderC()
    _lib.check(_lib.load().isort_sequence_read_header(os.fsencode(path), ctypes.byref(h)))
    return _hdr(h)


def load(path: str | os.PathLike, key_bytes: int = 4, device=None):
    """Keys of `path` in a new device tensor (int32 / int64 bit patterns of u32 / u64)."""
    import torch

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    hdr = read_header(path)
    keys = torch.empty(hdr.n, dtype=torch.int32 if key_bytes == 4 else torch.int64, device=dev)
    h = _lib.SequenceHeaderC()
    torch.cuda.synchronize(dev)
    _lib.check(_lib.load().isort_sequence_load(os.fsencode(path), keys.data_ptr() if hdr.n else None, hdr.n,
                                               key_bytes, ctypes.byref(h), dev.index))
    return _hdr(h), keys


def read_sequence(path: str | os.PathLike, device=None):
    """read_sequence_file: (header, records) with tag = position, keys via the device loader."""
    from .intsort import RECORD_DTYPE

    hdr, keys = load(path, key_bytes=8, device=device)
    rec = np.empty(hdr.n, dtype=RECORD_DTYPE)
    rec["key"] = keys.cpu().numpy().view(np.uint64)
    rec["tag"] = np.arange(hdr.n, dtype=np.uint64)
    return hdr, rec
