"""TNS1 tensor files and JSON reports.

The reference moves tensors between its CLI and other tools as TNS1 files
(src/core.py:93-152): a 16-byte little-endian header — magic b"TNS1",
version u32 = 1, dtype u8 (0 = f32, 1 = f64), rank u8 (1..3), reserved
u16 = 0 — then `rank` u64 extents and the row-major payload. Files written
here are byte-identical to the reference's for the same array, and every
malformed input raises the reference's error class (FormatError for the
header, LengthError for a short / long payload, ShapeError for non-finite
data), so GPU and CPU runs can be cross-checked through files.
"""

from __future__ import annotations

import json
import os
import struct
from dataclasses import dataclass, field

import numpy as np

from .core import FormatError, LengthError, ShapeError

_HDR = struct.Struct("<4sIBBH")
_CODES = {0: np.dtype("<f4"), 1: np.dtype("<f8")}


@dataclass
class Tensor:
    """Rank 1..3 row-major f32/f64 array, finite everywhere (the reference's
    validated carrier, src/core.py:48-90); rank 3 is [head, position, dim]."""

    array: np.ndarray

    def __post_init__(self):
        a = np.asarray(self.array)
        if a.dtype not in (np.float32, np.float64):
            raise ShapeError(f"dtype must be float32 or float64, got {a.dtype}")
        if not 1 <= a.ndim <= 3:
            raise ShapeError(f"rank must be 1..3, got {a.ndim}")
        if a.size == 0 or min(a.shape) < 1:
            raise ShapeError(f"all extents must be >= 1, got {a.shape}")
        if not np.all(np.isfinite(a)):
            raise ShapeError("tensor contains non-finite values")
        self.array = np.ascontiguousarray(a)

    @property
    def dims(self) -> tuple:
        return tuple(int(x) for x in self.array.shape)


def tensor_write(t, path) -> None:
    """Write a TNS1 file atomically (temp file + rename)."""
    if not isinstance(t, Tensor):
        t = Tensor(np.asarray(t))
    a = t.array
    code = 0 if a.dtype == np.float32 else 1
    blob = _HDR.pack(b"TNS1", 1, code, a.ndim, 0) + np.asarray(a.shape, dtype="<u8").tobytes() + \
        np.ascontiguousarray(a, dtype=_CODES[code]).tobytes()
    tmp = f"{path}.tmp.{os.getpid()}"
    try:
        with open(tmp, "wb") as fh:
            fh.write(blob)
        os.replace(tmp, path)
    except OSError:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def tensor_read(path) -> Tensor:
    """Read a TNS1 file (the exact inverse of tensor_write)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < _HDR.size:
        raise LengthError(f"{len(blob)} bytes: shorter than the {_HDR.size}-byte header")
    magic, version, code, rank, reserved = _HDR.unpack_from(blob)
    if magic != b"TNS1":
        raise FormatError(f"bad magic {magic!r}")
    if version != 1:
        raise FormatError(f"unsupported version {version}")
    if code not in _CODES:
        raise FormatError(f"unknown dtype code {code}")
    if not 1 <= rank <= 3:
        raise FormatError(f"rank must be 1..3, got {rank}")
    if reserved != 0:
        raise FormatError(f"reserved field must be 0, got {reserved}")
    end = _HDR.size + 8 * rank
    if len(blob) < end:
        raise LengthError("file ends inside the extents table")
    dims = [int(x) for x in np.frombuffer(blob, dtype="<u8", count=rank, offset=_HDR.size)]
    if min(dims) < 1:
        raise FormatError(f"all extents must be >= 1, got {dims}")
    dt = _CODES[code]
    n = int(np.prod(dims))
    if len(blob) != end + n * dt.itemsize:
        raise LengthError(f"payload is {len(blob) - end} bytes, expected {n * dt.itemsize}")
    arr = np.frombuffer(blob, dtype=dt, count=n, offset=end).reshape(dims).astype(dt.newbyteorder("="))
    try:
        return Tensor(arr)
    except ShapeError as exc:
        raise FormatError(str(exc)) from exc


@dataclass
class RunReport:
    """One command's outcome; to_json() validates against the reference's
    report schema (src/report_schema.json:1-22: command, config, metrics of
    numbers / number lists, pass, version)."""

    command: str
    config: dict
    metrics: dict = field(default_factory=dict)
    passed: bool = False

    def to_dict(self) -> dict:
        from . import __version__
        return {"command": self.command, "config": self.config, "metrics": self.metrics, "pass": self.passed,
                "version": __version__}

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), indent=2, allow_nan=False)


def write_json_atomic(obj, path) -> None:
    tmp = f"{path}.tmp.{os.getpid()}"
    try:
        with open(tmp, "w") as fh:
            json.dump(obj, fh, indent=2, allow_nan=False)
        os.replace(tmp, path)
    except OSError:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise
