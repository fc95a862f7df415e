"""Batched standalone transforms (cfg5 throughput): per-polynomial device
time of ntt_ct and intt_gs (scaled) over a batch of 1024 polynomials
(capped at 2^27 words), CUDA events around 10 back-to-back calls, median of
7 repetitions, and the CT-butterfly rate (n/2 log2 n butterflies per
forward transform).  Polynomial 0 of each batch is checked against the C
oracle.  Use NTTMUL_LIB to compare library builds.

    python scripts/batched_xform.py [--min-log 13] [--max-log 17]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (checker only)
import paper_2209_01290_b200 as nt  # noqa: E402


def per_call_ms(fn, calls=10, reps=7):
    s = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(calls):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / calls)
    return sorted(out)[reps // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-log", type=int, default=13)
    ap.add_argument("--max-log", type=int, default=17)
    args = ap.parse_args()
    for log_n in range(args.min_log, args.max_log + 1):
        n = 1 << log_n
        batch = min(1024, (1 << 27) // n)
        plan = nt.build_plan(n, bits=60, seed=0)
        rng = np.random.default_rng(log_n)
        x0 = rng.integers(0, plan.q, n, dtype=np.uint64)
        x = torch.from_numpy(np.broadcast_to(x0, (batch, n)).copy()).cuda()
        nt.kernels.ntt_ct(x, plan.tw_fwd, *plan.red_args, False, None)
        f, _ = oracle.twiddles(plan.q, plan.psi, log_n)
        w = x0.copy()
        oracle.ntt_ct(w, f, *plan.red_args, False)
        ok = bool(np.array_equal(x[0].cpu().numpy(), w))
        nt.kernels.intt_gs(x, plan.tw_inv, plan.q, (plan.q + 1) // 2, *plan.red_args[1:], True,
                           False, None)
        ok = ok and bool(np.array_equal(x[-1].cpu().numpy(), x0))
        fwd = per_call_ms(lambda: nt.kernels.ntt_ct(x, plan.tw_fwd, *plan.red_args, False, None))
        inv = per_call_ms(lambda: nt.kernels.intt_gs(x, plan.tw_inv, plan.q, (plan.q + 1) // 2,
                                                     *plan.red_args[1:], True, False, None))
        bfly = n // 2 * log_n
        print(json.dumps({
            "log_n": log_n, "batch": batch, "parity": ok,
            "ntt_us_per_poly": round(1e3 * fwd / batch, 4),
            "intt_us_per_poly": round(1e3 * inv / batch, 4),
            "ntt_gbfly_s": round(bfly * batch / (fwd * 1e-3) / 1e9, 1),
            "intt_gbfly_s": round(bfly * batch / (inv * 1e-3) / 1e9, 1),
            "lib": os.environ.get("NTTMUL_LIB", "default")}), flush=True)


if __name__ == "__main__":
    main()
