"""OMNT binary tensor files (reference ``tensorfile.py:1-54``).

Layout: 4-byte magic ``b"OMNT"``, little-endian u32 version (1), u64 rows,
u64 cols, then rows x cols little-endian float64 values, row-major. Writes go
to a sibling temporary file that is fsync'ed and renamed over the target, so
readers never see a partial file; a save/load round trip is bit-exact.
Non-finite values are refused on both sides, as in the reference.
"""

from __future__ import annotations

import os
import struct
from pathlib import Path

import numpy as np

from .errors import TensorFileError

MAGIC = b"OMNT"
VERSION = 1
HEADER = struct.Struct("<4sIQQ")  # magic, version, rows, cols (24 bytes)


def save_tensor(path, tensor) -> None:
    """Write a 2-D matrix (anything array-like, incl. CPU/GPU torch tensors)."""
    if hasattr(tensor, "detach"):
        tensor = tensor.detach().to("cpu").double().numpy()
    m = np.asarray(tensor, dtype=np.float64)
    if m.ndim != 2:
        raise TensorFileError(f"OMNT holds 2-D matrices; got {m.ndim} dimensions")
    if not np.all(np.isfinite(m)):
        raise TensorFileError("non-finite values cannot be stored")
    target = Path(path)
    tmp = target.parent / (target.name + ".tmp")
    payload = np.ascontiguousarray(m).astype("<f8", copy=False).tobytes()
    with open(tmp, "wb") as fh:
        fh.write(HEADER.pack(MAGIC, VERSION, m.shape[0], m.shape[1]))
        fh.write(payload)
        fh.flush()
        os.fsync(fh.fileno())
    os.replace(tmp, target)


def load_tensor(path) -> np.ndarray:
    """Read a matrix written by :func:`save_tensor` (or the reference)."""
    raw = Path(path).read_bytes()
    if len(raw) < HEADER.size:
        raise TensorFileError(f"{path}: file shorter than the 24-byte header")
    magic, version, rows, cols = HEADER.unpack_from(raw)
    if magic != MAGIC:
        raise TensorFileError(f"{path}: magic {magic!r} is not {MAGIC!r}")
    if version != VERSION:
        raise TensorFileError(f"{path}: version {version} not supported")
    body = raw[HEADER.size:]
    if len(body) != rows * cols * 8:
        raise TensorFileError(f"{path}: {len(body)} payload bytes, header says {rows} x {cols} float64")
    m = np.frombuffer(body, dtype="<f8").reshape(rows, cols).astype(np.float64)
    if not np.all(np.isfinite(m)):
        raise TensorFileError(f"{path}: payload holds non-finite values")
    return m
