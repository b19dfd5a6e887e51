"""KVQD tensor dumps (reference proj/include/kivi/dump_io.hpp, src/dump_io.cpp):
the reference's on-disk format for K/V tensors, used here to export materialised
device caches (parity artefacts, analysis ingestion).

Format (dump_io.hpp:10-17, little-endian):
    magic "KVQD" | version u32 = 1 | dtype u8 = 0 (float32) | ndim u8 in {1,2,3}
    | dims ndim x u64 | payload row-major float32
1-D loads as one 1 x n matrix, 2-D as one matrix, 3-D (heads x tokens x dim) as
one matrix per head.  Errors carry the byte offset, as the reference's do.
"""
from __future__ import annotations

import struct

import numpy as np

from . import FormatError, ShapeError, UsageError

MAGIC = b"KVQD"
VERSION = 1


def read_dump(path: str) -> list:
    """reference read_dump (dump_io.cpp:23-76): list of float32 [rows, cols] arrays."""
    try:
        f = open(path, "rb")
    except OSError:
        raise FormatError(f"cannot open dump file {path}", 0)
    with f:
        buf = f.read()
    if len(buf) < 4 or buf[:4] != MAGIC:
        raise FormatError('bad magic, expected "KVQD"', 0)

    def field(off, fmt, what):
        n = struct.calcsize(fmt)
        if len(buf) < off + n:
            raise FormatError(f"truncated dump file while reading {what}", off)
        return struct.unpack_from(fmt, buf, off)[0]

    version = field(4, "<I", "version")
    if version != VERSION:
        raise FormatError(f"unsupported version {version}", 4)
    dtype = field(8, "<B", "dtype")
    if dtype != 0:
        raise FormatError(f"unsupported dtype {dtype}", 8)
    ndim = field(9, "<B", "ndim")
    if not 1 <= ndim <= 3:
        raise FormatError("ndim must be 1, 2 or 3", 9)
    dims, off = [], 10
    for _ in range(ndim):
        dims.append(field(off, "<Q", "dims"))
        off += 8
    if ndim == 1:
        heads, rows, cols = 1, 1, dims[0]
    elif ndim == 2:
        heads, rows, cols = 1, dims[0], dims[1]
    else:
        heads, rows, cols = dims
    out = []
    nbytes = rows * cols * 4
    for h in range(heads):
        start = off + h * nbytes
        if len(buf) < start + nbytes:
            raise FormatError("truncated payload", start + max(0, len(buf) - start))
        m = np.frombuffer(buf, "<f4", rows * cols, start).reshape(rows, cols).copy()
        if not np.all(np.isfinite(m)):
            raise UsageError(f"read_dump({path}): non-finite value in {rows}x{cols} matrix")
        out.append(m)
    return out


def write_dump(path: str, tensors) -> None:
    """reference write_dump (dump_io.cpp:78-105): one tensor as 2-D, several
    same-shaped tensors as 3-D."""
    tensors = [np.ascontiguousarray(t, dtype="<f4") for t in tensors]
    if not tensors:
        raise UsageError("write_dump: no tensors")
    tensors = [t.reshape(1, -1) if t.ndim == 1 else t for t in tensors]
    if any(t.shape != tensors[0].shape for t in tensors):
        raise ShapeError("write_dump: tensors in one dump must share a shape")
    rows, cols = tensors[0].shape
    ndim = 2 if len(tensors) == 1 else 3
    dims = (rows, cols) if ndim == 2 else (len(tensors), rows, cols)
    try:
        with open(path, "wb") as f:
            f.write(MAGIC + struct.pack("<IBB", VERSION, 0, ndim))
            f.write(struct.pack(f"<{ndim}Q", *dims))
            for t in tensors:
                f.write(t.tobytes())
    except OSError:
        raise UsageError(f"write_dump: cannot open {path}")


def export_cache_unit(cache, unit: int, key_path: str, value_path: str) -> None:
    """Materialise one unit of a device cache (reference materialize_keys /
    materialize_values, kv_cache.cpp:100-106, run on the GPU) and dump K and V."""
    k, v = cache.materialize()
    write_dump(key_path, [k[unit].cpu().numpy()])
    write_dump(value_path, [v[unit].cpu().numpy()])
