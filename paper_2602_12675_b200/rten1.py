"""RTEN1 tensor files: the reference's golden-exchange format (tensor_io.hpp:12-115).

    magic "RTEN1\\0" | u32le rank | u32le dims[rank] | u8 dtype (0 = f32, 1 = f64) | raw LE data

`save` / `load` read and write it from numpy arrays (any rank, float32 / float64), raising
ContractError with the reference's messages on a bad magic, a dtype mismatch or a truncated
file (tensor_io.hpp:60-78). `save_matrix` / `load_matrix` and `save_vector` / `load_vector`
mirror sla2::rten::save / load_matrix / load_vector (rank 2 / rank 1). The parity harness uses
them to exchange inputs and outputs with the reference (tests/test_rten1.py,
tests/golden/rten1/)."""
from __future__ import annotations

import os
import struct

import numpy as np

MAGIC = b"RTEN1\x00"
_CODES = {np.dtype(np.float32): 0, np.dtype(np.float64): 1}
_DTYPES = {0: np.dtype("<f4"), 1: np.dtype("<f8")}


def _contract(msg):
    from . import ContractError  # the package's exception for the reference's contract_error
    return ContractError(msg)


def save(path: str | os.PathLike, array) -> None:
    a = np.asarray(array)
    if a.dtype not in _CODES:
        raise _contract("RTEN1 supports f32 and f64 only")  # tensor_io.hpp:20-22
    try:
        f = open(path, "wb")
    except OSError:
        raise _contract(f"RTEN1: cannot open for write: {path}") from None
    with f:
        f.write(MAGIC)
        f.write(struct.pack("<I", a.ndim))
        f.write(struct.pack(f"<{a.ndim}I", *a.shape))
        f.write(struct.pack("<B", _CODES[a.dtype]))
        f.write(np.ascontiguousarray(a, dtype=a.dtype.newbyteorder("<")).tobytes())


def load(path: str | os.PathLike, dtype=None) -> np.ndarray:
    """Any-rank read. With `dtype` given, a file of the other dtype is a contract error, as in
    the reference's typed loaders (tensor_io.hpp:73-75)."""
    try:
        f = open(path, "rb")
    except OSError:
        raise _contract(f"RTEN1: cannot open: {path}") from None
    with f:
        buf = f.read()
    if len(buf) < 11 or buf[:6] != MAGIC:
        raise _contract(f"RTEN1: bad magic in {path}")
    rank = struct.unpack_from("<I", buf, 6)[0]
    off = 10
    if len(buf) < off + 4 * rank + 1:
        raise _contract(f"RTEN1: truncated file {path}")
    dims = struct.unpack_from(f"<{rank}I", buf, off)
    off += 4 * rank
    code = buf[off]
    off += 1
    if code not in _DTYPES or (dtype is not None and _CODES.get(np.dtype(dtype)) != code):
        raise _contract(f"RTEN1: dtype mismatch in {path}")
    dt = _DTYPES[code]
    count = int(np.prod(dims, dtype=np.int64)) if rank else 1
    if len(buf) - off < count * dt.itemsize:
        raise _contract(f"RTEN1: truncated file {path}")
    return np.frombuffer(buf, dtype=dt, count=count, offset=off).reshape(dims).astype(dt.newbyteorder("="))


def save_matrix(path, m) -> None:
    m = np.asarray(m)
    if m.ndim != 2:
        raise _contract("RTEN1: expected rank 2")
    save(path, m)


def save_vector(path, v) -> None:
    v = np.asarray(v)
    if v.ndim != 1:
        raise _contract("RTEN1: expected rank 1")
    save(path, v)


def load_matrix(path, dtype=np.float32) -> np.ndarray:
    a = load(path, dtype)
    if a.ndim != 2:
        raise _contract(f"RTEN1: expected rank 2 in {path}")  # tensor_io.hpp:101
    return a


def load_vector(path, dtype=np.float32) -> np.ndarray:
    a = load(path, dtype)
    if a.ndim != 1:
        raise _contract(f"RTEN1: expected rank 1 in {path}")  # tensor_io.hpp:111
    return a
