"""FCTN tensor / mask containers and reports — the reference's file formats
(`fctnlr.fileio`, fileio.py:1-120), so files move between the two tools.

Container (little-endian): magic ``FCTN``, format version u32 (1), element
code u32 (1 = float64, 2 = mask byte), order u32, one u64 extent per mode,
then the payload first-index-fastest; mask bytes strictly 0 or 1
(fileio.py:1-8, 59-120).  Writes go through a temp file in the target
directory and an atomic rename (fileio.py:40-55).  Same ValueError messages
for malformed input.  `sample_mask` is the reference's exact-count sampler
(fileio.py:123-136; implemented in workloads.py).
"""
from __future__ import annotations

import csv
import io
import os
import struct
import tempfile

import numpy as np

from .workloads import sample_mask

__all__ = ["MAGIC", "read_mask", "read_tensor", "sample_mask", "write_mask", "write_report_csv", "write_tensor"]

MAGIC = b"FCTN"
FORMAT_VERSION = 1
ELEM_F64 = 1
ELEM_MASK = 2
_HEADER = struct.Struct("<4sIII")


def _atomic_write(path: str, chunks) -> None:
    directory = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(prefix=".fctn-", dir=directory)
    try:
        with os.fdopen(fd, "wb") as fh:
            for c in chunks:
                fh.write(c)
            fh.flush()
            os.fsync(fh.fileno())
        os.replace(tmp, path)
    except BaseException:
        try:
            os.unlink(tmp)
        except OSError:
            pass
        raise


def _header(shape, elem: int) -> bytes:
    return _HEADER.pack(MAGIC, FORMAT_VERSION, elem, len(shape)) + struct.pack(f"<{len(shape)}Q", *shape)


def _parse(blob: memoryview, path: str):
    if len(blob) < _HEADER.size:
        raise ValueError(f"{path}: truncated header")
    magic, version, elem, order = _HEADER.unpack_from(blob, 0)
    if magic != MAGIC:
        raise ValueError(f"{path}: bad magic {magic!r}")
    if version != FORMAT_VERSION:
        raise ValueError(f"{path}: unsupported format version {version}")
    if order < 1:
        raise ValueError(f"{path}: order must be >= 1")
    need = _HEADER.size + 8 * order
    if len(blob) < need:
        raise ValueError(f"{path}: truncated extent list")
    extents = struct.unpack_from(f"<{order}Q", blob, _HEADER.size)
    if any(e < 1 for e in extents):
        raise ValueError(f"{path}: zero extent")
    return elem, tuple(int(e) for e in extents), blob[need:]


def _read(path: str):
    with open(path, "rb") as fh:
        return memoryview(fh.read())


def write_tensor(path: str, arr: np.ndarray) -> None:
    """float64 container (fileio.py:82-87); the payload is written straight
    from the F-order buffer (no byte-string copy of a multi-GB tensor)."""
    arr = np.asarray(arr, dtype=np.float64)
    if arr.ndim < 1:
        arr = arr.reshape(1)
    f = np.asfortranarray(arr).astype("<f8", copy=False)
    _atomic_write(path, [_header(arr.shape, ELEM_F64), memoryview(f.reshape(-1, order="F")).cast("B")])


def read_tensor(path: str) -> np.ndarray:
    elem, extents, payload = _parse(_read(path), path)
    if elem != ELEM_F64:
        raise ValueError(f"{path}: element code {elem} is not a float64 tensor")
    count = int(np.prod(extents, dtype=np.int64))
    if len(payload) != 8 * count:
        raise ValueError(f"{path}: payload has {len(payload)} bytes, expected {8 * count}")
    return np.frombuffer(payload, dtype="<f8").astype(np.float64).reshape(extents, order="F")


def write_mask(path: str, mask: np.ndarray) -> None:
    mask = np.asarray(mask, dtype=bool)
    if mask.ndim < 1:
        mask = mask.reshape(1)
    payload = np.asfortranarray(mask).view(np.uint8).reshape(-1, order="F")
    _atomic_write(path, [_header(mask.shape, ELEM_MASK), memoryview(np.ascontiguousarray(payload)).cast("B")])


def read_mask(path: str) -> np.ndarray:
    elem, extents, payload = _parse(_read(path), path)
    if elem != ELEM_MASK:
        raise ValueError(f"{path}: element code {elem} is not a mask")
    count = int(np.prod(extents, dtype=np.int64))
    if len(payload) != count:
        raise ValueError(f"{path}: payload has {len(payload)} bytes, expected {count}")
    flat = np.frombuffer(payload, dtype=np.uint8)
    if flat.size and int(flat.max()) > 1:
        raise ValueError(f"{path}: mask bytes must be strictly 0 or 1")
    return flat.astype(bool).reshape(extents, order="F")


def write_report_csv(path: str, rows, fieldnames) -> None:
    """Per-iteration trace CSV (fileio.py:139-146)."""
    buf = io.StringIO()
    writer = csv.DictWriter(buf, fieldnames=list(fieldnames), lineterminator="\n")
    writer.writeheader()
    for row in rows:
        writer.writerow(row)
    _atomic_write(path, [buf.getvalue().encode("utf-8")])
