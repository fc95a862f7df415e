"""Polynomial file formats of the reference front end (cli.py:57-125).

* binary ``NTTP`` v1: magic ``b"NTTP"``, version byte 1, n and q as
  little-endian uint64, then n little-endian uint64 coefficients;
* text: a header line ``"n q"`` then one coefficient per line.

The byte layouts, validation and error messages (with the offending line
number) are the reference's, so files written by either package read back
in the other.  Binary payloads move as one numpy buffer (no per-coefficient
Python work) and can be loaded straight into a CUDA tensor.
"""

from __future__ import annotations

import numpy as np

_BIN_MAGIC = b"NTTP"
_BIN_VERSION = 1


class InputError(Exception):
    """Bad input file or inconsistent arguments (the CLI's exit code 2)."""


def write_poly(path: str, coeffs, n: int, q: int, binary: bool) -> None:
    """Write n coefficients (mod q) in the binary or text format."""
    if binary:
        body = np.asarray(coeffs, dtype="<u8")
        if body.size != n:
            raise InputError(f"{path}: {body.size} coefficients for n={n}")
        with open(path, "wb") as fh:
            fh.write(_BIN_MAGIC)
            fh.write(bytes([_BIN_VERSION]))
            fh.write(int(n).to_bytes(8, "little"))
            fh.write(int(q).to_bytes(8, "little"))
            fh.write(body.tobytes())
    else:
        with open(path, "w") as fh:
            fh.write(f"{n} {q}\n")
            for c in np.asarray(coeffs).tolist():
                fh.write(f"{int(c)}\n")


def read_poly(path: str, binary: bool) -> tuple[int, int, np.ndarray]:
    """(n, q, coefficients as uint64[n]); raises InputError with the
    offending line number on malformed text input."""
    if binary:
        with open(path, "rb") as fh:
            data = fh.read()
        if data[:4] != _BIN_MAGIC:
            raise InputError(f"{path}: bad magic, not a binary polynomial file")
        if len(data) < 21:
            raise InputError(f"{path}: truncated header")
        if data[4] != _BIN_VERSION:
            raise InputError(f"{path}: unsupported version {data[4]}")
        n = int.from_bytes(data[5:13], "little")
        q = int.from_bytes(data[13:21], "little")
        body = data[21:]
        if len(body) != 8 * n:
            raise InputError(f"{path}: expected {8 * n} payload bytes, got {len(body)}")
        return n, q, np.frombuffer(body, dtype="<u8").astype(np.uint64)
    with open(path) as fh:
        lines = fh.read().splitlines()
    if not lines:
        raise InputError(f"{path}:1: empty file")
    head = lines[0].split()
    if len(head) != 2:
        raise InputError(f"{path}:1: expected header 'n q'")
    try:
        n, q = int(head[0]), int(head[1])
    except ValueError:
        raise InputError(f"{path}:1: non-integer header") from None
    if len(lines) < n + 1:
        raise InputError(f"{path}: expected {n} coefficient lines, got {len(lines) - 1}")
    coeffs = np.empty(n, dtype=np.uint64)
    for i in range(n):
        try:
            c = int(lines[1 + i])
        except ValueError:
            raise InputError(f"{path}:{i + 2}: non-integer coefficient") from None
        if not 0 <= c < q:
            raise InputError(f"{path}:{i + 2}: coefficient {c} outside [0, q)")
        coeffs[i] = c
    return n, q, coeffs
