"""The reference's bench CSV contract (reference cli.py:47-55, 213-325) with
GPU timings.

One row per (kernel, n, bits, variant): ``CSV_HEADER`` = kernel, n, bits,
variant, reps, min/mean/median nanoseconds per call, and the OpCounter tallies
of ONE call (modmul, addsub, half, twiddle_loads).  The kernels, their
operands (``Polynomial.random`` on a ``random.Random(seed)`` stream, a fixed
4096-entry block for the reduction kernels) and the counting follow the
reference's ``_bench_reduction`` / ``_bench_transform`` / ``cmd_bench``; the
calls run on the GPU through this package's public API, and each timed call
is bracketed by ``torch.cuda.synchronize()`` so the time is the call's full
latency as the host sees it (the reference times a blocking CPU call).  The
reduction kernels report time per reduction, like the reference.

    python -m paper_2209_01290_b200.benchcsv --kernel polymul-fused --n 65536 \\
        --bits 60 [--csv out.csv]

The command-line parsing of the reference (``nttmul bench`` and its other
sub-commands) is out of scope; this module keeps only its output contract.
"""

from __future__ import annotations

import argparse
import csv
import os
import random
import statistics
import sys
import time

import numpy as np
import torch

from . import kernels
from .modarith import Modulus
from .nttcore import OpCounter, Polynomial, batch_ntt, intt_gs_scaled, ntt_2d, ntt_ct, \
    ntt_radix4
from .params import build_plan
from .polymul import FusedPlan, polymul_fused, polymul_ntt

BENCH_KERNELS = (
    "reduce-builtin", "barrett-classical", "barrett-dhem", "barrett-proposed",
    "ntt", "intt", "ntt-radix4", "ntt-2d", "polymul", "polymul-fused",
    "batch-ntt",
)

CSV_HEADER = ("kernel", "n", "bits", "variant", "reps",
              "min_ns", "mean_ns", "median_ns",
              "modmul", "addsub", "half", "twiddle_loads")

_REDUCTION_VARIANT = {"reduce-builtin": "builtin", "barrett-classical": "classical",
                      "barrett-dhem": "dhem", "barrett-proposed": "proposed"}


def _time_samples(fn, reps: int, warmup: int) -> list[int]:
    """Per-call latencies in nanoseconds (reference cli.py:213-222), each
    call synchronised with the device on both sides."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        t0 = time.perf_counter_ns()
        fn()
        torch.cuda.synchronize()
        out.append(time.perf_counter_ns() - t0)
    return out


def _bench_reduction(kernel: str, bits: int, reps: int, warmup: int, seed: int):
    """Per-reduction latency via the mulmod loop over a fixed 4096-entry
    block (reference cli.py:225-248)."""
    variant = _REDUCTION_VARIANT[kernel]
    rng = random.Random(seed)
    q = build_plan(2, bits=bits, seed=seed).q
    mode, mu, s_in, s_out = Modulus(q).reduction_params(variant)
    block = 4096
    a = np.array([rng.randrange(q) for _ in range(block)], dtype=np.uint64)
    b = np.array([rng.randrange(q) for _ in range(block)], dtype=np.uint64)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    chunks = max(1, reps // block)

    def one():
        kernels.mulmod_loop(da, db, q, mode, mu, s_in, s_out, 1)

    times = _time_samples(one, chunks, max(1, warmup // block))
    per_op = [t / block for t in times]
    return q, variant, chunks * block, per_op, OpCounter(modmul=chunks * block)


def _bench_transform(kernel: str, n: int, bits: int, reps: int, warmup: int,
                     workers: int, seed: int, variant: str):
    """One transform / product per call on the reference's operands
    (reference cli.py:251-297); the counts are those of one call."""
    plan = build_plan(n, bits=bits, seed=seed, variant=variant)
    rng = random.Random(seed)
    base = Polynomial.random(plan, rng)
    ctr = OpCounter()
    if kernel in ("ntt", "ntt-radix4", "ntt-2d"):
        fwd = {"ntt": ntt_ct, "ntt-radix4": ntt_radix4, "ntt-2d": ntt_2d}[kernel]
        fwd(base.copy(), plan, ctr)

        def one():
            fwd(base.copy(), plan)
    elif kernel == "intt":
        spec = ntt_ct(base.copy(), plan)
        intt_gs_scaled(spec.copy(), plan, ctr)

        def one():
            intt_gs_scaled(spec.copy(), plan)
    elif kernel in ("polymul", "polymul-fused"):
        b2 = Polynomial.random(plan, rng)
        if kernel == "polymul":
            def fn(c=None):
                return polymul_ntt(base.coeffs, b2.coeffs, plan, c)
        else:
            fused = FusedPlan.from_plan(plan)

            def fn(c=None):
                return polymul_fused(base.coeffs, b2.coeffs, fused, c)
        fn(ctr)

        def one():
            fn()
    elif kernel == "batch-ntt":
        nrows = max(8, 4 * workers)
        rows = [Polynomial.random(plan, rng) for _ in range(nrows)]
        batch_ntt([r.copy() for r in rows], plan, workers, ctr)

        def one():
            batch_ntt([r.copy() for r in rows], plan, workers)
    else:
        raise ValueError(f"unknown bench kernel {kernel!r}")
    times = _time_samples(one, reps, warmup)
    return plan.q, variant, reps, times, ctr


def bench_row(kernel: str, n: int = 4096, bits: int = 60, reps: int = 20, warmup: int = 3,
              workers: int = 1, seed: int = 0, variant: str = "proposed") -> tuple:
    """One CSV row in CSV_HEADER order (reference cmd_bench, cli.py:300-316)."""
    if kernel not in BENCH_KERNELS:
        raise ValueError(f"unknown bench kernel {kernel!r}")
    if kernel.startswith(("reduce", "barrett")):
        _, variant, reps, times, ctr = _bench_reduction(kernel, bits, reps, warmup, seed)
        n = 1
    else:
        _, variant, reps, times, ctr = _bench_transform(kernel, n, bits, reps, warmup,
                                                        workers, seed, variant)
    return (kernel, n, bits, variant, reps,
            round(min(times), 1), round(statistics.fmean(times), 1),
            round(statistics.median(times), 1),
            ctr.modmul, ctr.modadd_sub, ctr.half_scalings, ctr.twiddle_loads)


def write_row(row, path: str | None = None) -> None:
    """Append to ``path`` (header first when the file is new or empty), or
    print header + row to stdout (reference cli.py:317-325)."""
    if path:
        fresh = not (os.path.exists(path) and os.path.getsize(path))
        with open(path, "a", newline="") as fh:
            w = csv.writer(fh)
            if fresh:
                w.writerow(CSV_HEADER)
            w.writerow(row)
    else:
        w = csv.writer(sys.stdout)
        w.writerow(CSV_HEADER)
        w.writerow(row)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--kernel", required=True, choices=BENCH_KERNELS)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--bits", type=int, default=60)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--variant", default="proposed")
    ap.add_argument("--csv", default=None)
    a = ap.parse_args(argv)
    write_row(bench_row(a.kernel, a.n, a.bits, a.reps, a.warmup, a.workers, a.seed, a.variant),
              a.csv)
    return 0


if __name__ == "__main__":
    sys.exit(main())
