"""SNGD binary datasets and label files (the data format
on the input side of the hot path).

Same layout, names, messages and error types as the reference:
  binary layout      proj/include/sng/io.hpp:28-31 -- magic "SNGD", version byte
                     1, little-endian u64 n and dim, then n*dim little-endian
                     IEEE doubles, row-major
  save/load_binary   proj/src/io.cpp:123-155
  load_points        proj/src/io.cpp:157-166 (binary by magic; the CSV reader is
                     out of scope here and raises NotImplementedError)
  save/load_labels   proj/src/io.cpp:168-193 -- one integer per line, noise "-1"
  ParseError/IoError proj/include/sng/errors.hpp

`load_binary` returns the reference's fp64 rows as a Dataset: rows that fp32
holds exactly go to the device as fp32, others take the exact fp64 entry
points (Dataset.values64), so a file goes straight to the GPU path.
"""
from __future__ import annotations

import struct

import numpy as np

from . import Clustering, Dataset

MAGIC = b"SNGD"
VERSION = 1
_HEADER = struct.Struct("<4sBQQ")  # magic, version, n, dim (packed: 21 bytes)


class ParseError(RuntimeError):
    """Malformed input; carries the 1-based line number when one applies."""

    def __init__(self, message: str, line: int = 0):
        super().__init__(f"line {line}: {message}" if line > 0 else message)
        self.line = line


class IoError(RuntimeError):
    """Filesystem-level failure (missing file, unwritable path, truncated stream)."""


def save_binary(data: Dataset, path: str) -> None:
    vals = data.values64 if data.values64 is not None else data.values.astype(np.float64)
    n, dim = vals.shape
    try:
        with open(path, "wb") as f:
            f.write(_HEADER.pack(MAGIC, VERSION, n, dim))
            f.write(np.ascontiguousarray(vals, "<f8").tobytes())
    except OSError as e:
        raise IoError(f"error while writing '{path}'") from e


def load_binary(path: str) -> Dataset:
    try:
        f = open(path, "rb")
    except OSError as e:
        raise IoError(f"cannot open '{path}' for reading") from e
    with f:
        head = f.read(5)
        if len(head) < 4 or head[:4] != MAGIC:
            raise ParseError(f"file '{path}' is not an SNGD binary dataset")
        if len(head) < 5 or head[4] != VERSION:
            raise ParseError(f"unsupported SNGD version {head[4] if len(head) > 4 else -1}")
        dims = f.read(16)
        if len(dims) < 16:
            raise ParseError(f"corrupt SNGD header in '{path}'")
        n, dim = struct.unpack("<QQ", dims)
        if n == 0 or dim == 0:
            raise ParseError(f"corrupt SNGD header in '{path}'")
        payload = f.read(n * dim * 8)
        if len(payload) < n * dim * 8:
            raise ParseError(f"truncated SNGD payload in '{path}'")
    vals = np.frombuffer(payload, "<f8").astype(np.float64).reshape(n, dim)
    return Dataset(vals)


def load_points(path: str) -> Dataset:
    """Reads the binary format (decided by the 4-byte magic, io.cpp:157-166)."""
    try:
        with open(path, "rb") as f:
            magic = f.read(4)
    except OSError as e:
        raise IoError(f"cannot open '{path}' for reading") from e
    if magic == MAGIC:
        return load_binary(path)
    raise NotImplementedError("CSV datasets are outside this package's scope (SURVEY.md section 2)")


def save_labels(labels, path: str) -> None:
    try:
        with open(path, "w") as f:
            f.write("".join(f"{int(v)}\n" for v in np.asarray(labels, np.int32)))
    except OSError as e:
        raise IoError(f"cannot open '{path}' for writing") from e


def load_labels(path: str) -> np.ndarray:
    try:
        f = open(path)
    except OSError as e:
        raise IoError(f"cannot open '{path}' for reading") from e
    out = []
    with f:
        for line_no, line in enumerate(f, 1):
            line = line.rstrip("\n").rstrip("\r")
            if not line:
                continue
            try:
                v = int(line, 10)
            except ValueError:
                raise ParseError(f"label '{line}' is not an integer", line_no) from None
            if not -2**31 <= v < 2**31 or line.strip() != line or line[:1] == "+" or "_" in line:
                raise ParseError(f"label '{line}' is not an integer", line_no)
            out.append(v)
    return np.asarray(out, np.int32)


def save_clustering(c: Clustering, path: str) -> None:
    save_labels(c.assignment, path)


__all__ = ["MAGIC", "VERSION", "ParseError", "IoError", "save_binary", "load_binary",
           "load_points", "save_labels", "load_labels", "save_clustering"]
