"""File formats (reference dataio.py:1-108): fvecs vectors and the scalar
sidecar, plus re-exports of the GRAB v1 container and the synthetic generator.
Host-side file IO only (no compute)."""
from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .datasets import gen_synthetic
from .graph import load_index, save_index

__all__ = ["FvecsFormatError", "read_fvecs", "write_fvecs", "read_scalars", "write_scalars", "gen_synthetic",
           "load_index", "save_index"]


class FvecsFormatError(ValueError):
    """Malformed fvecs content; ``offset`` is the offending byte (dataio.py:18-23)."""

    def __init__(self, message: str, offset: int):
        super().__init__(f"{message} (byte offset {offset})")
        self.offset = offset


def read_fvecs(path) -> np.ndarray:
    """dataio.py:26-50: per record an i32 dimension then d little-endian f32."""
    raw = Path(path).read_bytes()
    if not raw:
        return np.zeros((0, 0), dtype=np.float32)
    if len(raw) < 4:
        raise FvecsFormatError("file shorter than one dimension header", 0)
    d = int(np.frombuffer(raw, dtype="<i4", count=1)[0])
    if d <= 0:
        raise FvecsFormatError(f"invalid dimension {d}", 0)
    rec = 4 + 4 * d
    if len(raw) % rec:
        raise FvecsFormatError(f"truncated record: file size {len(raw)} not a multiple of {rec}",
                               (len(raw) // rec) * rec)
    tab = np.frombuffer(raw, dtype="<i4").reshape(-1, d + 1)
    bad = np.flatnonzero(tab[:, 0] != d)
    if bad.size:
        raise FvecsFormatError(f"inconsistent dimension {tab[bad[0], 0]} (expected {d})", int(bad[0]) * rec)
    return tab[:, 1:].view("<f4").copy()


def write_fvecs(path, vectors) -> None:
    v = np.asarray(vectors, dtype="<f4")
    n, d = v.shape
    tab = np.empty((n, d + 1), dtype="<i4")
    tab[:, 0] = d
    tab[:, 1:] = v.view("<i4")
    Path(path).write_bytes(tab.tobytes())


def read_scalars(path) -> np.ndarray:
    """dataio.py:63-71: u64 count header, then that many little-endian f32."""
    raw = Path(path).read_bytes()
    if len(raw) < 8:
        raise ValueError(f"scalar sidecar too short: {len(raw)} bytes")
    (n,) = struct.unpack_from("<Q", raw, 0)
    if len(raw) != 8 + 4 * n:
        raise ValueError(f"scalar sidecar header says {n} values, file has {(len(raw) - 8) // 4}")
    return np.frombuffer(raw, dtype="<f4", count=n, offset=8).copy()


def write_scalars(path, scalars) -> None:
    s = np.asarray(scalars, dtype="<f4")
    with open(path, "wb") as f:
        f.write(struct.pack("<Q", len(s)))
        f.write(s.tobytes())
