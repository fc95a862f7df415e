"""Shared fixtures.  `-m gpu` tests need a B200 (sm_100a); everything else
runs on CPU (oracle vs golden vectors, host logic, C-ABI exports, gloo)."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def vectors():
    return dict(np.load(os.path.join(GOLDEN, "vectors.npz")))


def rand(q: int, n: int, seed: int) -> np.ndarray:
    """The golden generator's input recipe (tests/golden/make_golden.py)."""
    return np.random.default_rng(seed).integers(0, q, size=n, dtype=np.uint64)


def digest(a) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()
