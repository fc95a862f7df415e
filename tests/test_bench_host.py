"""bench.py host logic on CPU: the shard partition and config both arms
report, the algorithmic work counts behind `roofline`, the IMAD-pipe roof,
the committed per-kernel traffic, and that a limb shard's synthetic inputs
are exactly the whole job's rows (so per-rank parity checks and the
gathered product agree)."""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _args(**kw):
    base = dict(gpus=1, steps=20, warmup=5, impl="ours", batch=16, log_n=16, limbs=21,
                cpu_seconds=10.0, no_cpu_baseline=False, no_e2e=False, shard=None)
    base.update(kw)
    return argparse.Namespace(**base)


def test_shard_mode_defaults():
    assert bench.shard_mode(_args()) == "ct"
    assert bench.shard_mode(_args(log_n=17, limbs=32, batch=8)) == "limb"
    assert bench.shard_mode(_args(shard="limb")) == "limb"


def test_config_dict_both_arms():
    c = bench.config_dict(_args(gpus=8), 8)
    assert c["workload"].startswith("cfg3") and c["global_batch"] == 128
    assert c["batch_per_gpu"] == 16 and c["parallelism"] == "shard-by-ciphertext x8"
    c4 = bench.config_dict(_args(log_n=17, limbs=32, batch=8, gpus=8), 8)
    assert c4["workload"].startswith("cfg4") and c4["global_batch"] == 8
    assert c4["parallelism"] == "shard-by-limb x8" and c4["batch_per_gpu"] is None


def test_work_counts():
    # 33,718,272 modmuls per cfg3 ciphertext (21 limbs)
    assert 21 * bench.modmuls_per_product(1 << 16) == 33_718_272
    assert bench.modmuls_per_product(1 << 12) == 75_776
    n = 1 << 16  # row kernel: 2 (n/2) 11 + 2n + (n/2) 11, the columns 4n + 2n
    assert bench.row_kernel_modmuls(n) + 6 * n == bench.modmuls_per_product(n)


def test_imad_pipe_roof():
    r = bench.imad_pipe_roof(1 << 16, 1965.0)
    assert 30.0 < r["fmaheavy_cycles_per_modmul"] < 30.6
    assert 1200 < r["peak_gmodmul_s"] < 1260


def test_committed_traffic_covers_the_step():
    t = bench.load_traffic(336, 1 << 16)
    assert t is not None and t["complete"]
    assert set(t) >= {"col_fwd", "row_fused", "col_inv", "total", "ratio_to_24n"}
    assert 1.0 < t["ratio_to_24n"] < 4.0


def test_limb_shard_inputs_are_the_job_rows():
    primes = [1152921504606584833, 1152921504606748673, 1152921504606830593, 1152921504606748417]
    whole = bench.make_inputs(primes, 3, 64, seed=1000)
    for lo, hi in ((0, 2), (2, 4), (1, 3)):
        part = bench.make_inputs(primes[lo:hi], 3, 64, seed=1000, limb0=lo)
        assert np.array_equal(part, whole[:, lo:hi])
    assert all((whole[:, i] < q).all() for i, q in enumerate(primes))
