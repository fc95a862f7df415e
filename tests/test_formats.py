"""NTTP binary / text polynomial files: byte-compatible with the reference
(cli.py:57-125) in both directions, same validation errors (CPU only)."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2209_01290_b200 import formats


@pytest.mark.parametrize("binary", [True, False])
def test_roundtrip_and_reference_compat(tmp_path, binary):
    q = (1 << 60) - 93
    coeffs = np.random.default_rng(1).integers(0, q, 257, dtype=np.uint64)
    coeffs[:2] = [0, q - 1]
    p = str(tmp_path / "a.poly")
    formats.write_poly(p, coeffs, 257, q, binary)
    n, qq, got = formats.read_poly(p, binary)
    assert (n, qq) == (257, q) and np.array_equal(got, coeffs)
    ref = oracle.reference()
    if ref is not None:  # the reference reads ours and we read the reference's
        from nttmul import cli

        assert cli.read_poly(p, binary) == (257, q, [int(c) for c in coeffs])
        p2 = str(tmp_path / "b.poly")
        cli.write_poly(p2, [int(c) for c in coeffs], 257, q, binary)
        with open(p, "rb") as f1, open(p2, "rb") as f2:
            assert f1.read() == f2.read()


def test_errors(tmp_path):
    p = tmp_path / "x"
    p.write_bytes(b"XXXX\x01")
    with pytest.raises(formats.InputError, match="bad magic"):
        formats.read_poly(str(p), True)
    p.write_bytes(b"NTTP\x02" + (4).to_bytes(8, "little") + (97).to_bytes(8, "little"))
    with pytest.raises(formats.InputError, match="unsupported version 2"):
        formats.read_poly(str(p), True)
    p.write_bytes(b"NTTP\x01" + (4).to_bytes(8, "little") + (97).to_bytes(8, "little") + b"\0" * 8)
    with pytest.raises(formats.InputError, match="expected 32 payload bytes, got 8"):
        formats.read_poly(str(p), True)
    p.write_text("")
    with pytest.raises(formats.InputError, match=":1: empty file"):
        formats.read_poly(str(p), False)
    p.write_text("4 97\n1\n2\nx\n3\n")
    with pytest.raises(formats.InputError, match=":4: non-integer coefficient"):
        formats.read_poly(str(p), False)
    p.write_text("2 97\n1\n97\n")
    with pytest.raises(formats.InputError, match=r":3: coefficient 97 outside \[0, q\)"):
        formats.read_poly(str(p), False)
    p.write_text("3 97\n1\n")
    with pytest.raises(formats.InputError, match="expected 3 coefficient lines, got 1"):
        formats.read_poly(str(p), False)
