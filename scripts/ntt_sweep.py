"""BASELINE cfg5: Barrett-variant and radix-split sweep at N = 2^10 .. 2^17.

Standalone transforms through the reference-named kernel surface
(`kernels.ntt_ct` / `kernels.intt_gs`, reference _kernels.pyx:52-129):
latency with one polynomial and throughput with a batch of 1024 (capped at
2^27 coefficients), CUDA events on the launch stream, for

* every reduction variant (builtin / classical / dhem / proposed, reference
  modarith.py:73-82) at the default split - the transforms use Shoup
  twiddle products whatever the variant, the variant sets the data x data
  products (`mulmod_loop`, _kernels.pyx:359-371, reported per reduction);
* every radix split N1 x N2 the library offers for n > 4096
  (nttmul_set_split: rows of 2^10 .. 2^13 words, 1 .. 5 column stages) with
  the proposed variant, plus the fused product's rate at that split.

Every configuration is checked bit-exactly against the C oracle on
polynomial 0 before it is timed.  One JSON line per configuration.
``--ncu-plan`` instead runs each split configuration's batched forward
transform once, in order, for an ncu launch list (scripts/cfg5_ncu.py maps
the launches back to the configurations).

usage: python scripts/ntt_sweep.py [--out FILE] [--min-log 10] [--max-log 17]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (checker only)
import paper_2209_01290_b200 as nt  # noqa: E402

VARIANTS = ("builtin", "classical", "dhem", "proposed")
COL_LOG_R = 12  # default row length of the 2D split (ntt_kernels.cuh COL_LOG_R)


def splits(log_n):
    """Row lengths log2 N2 offered for this size (nttmul_set_split), default first."""
    if log_n <= COL_LOG_R:
        return [log_n]
    return [COL_LOG_R] + [r for r in (10, 11, 13) if 1 <= log_n - r <= 5]


def timed(fn, reps):
    stream = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps  # ms


def graph_us(fn, reps=20):
    """Device time per call from a CUDA graph of `reps` back-to-back calls
    (no host launch overhead); None if the calls cannot be captured."""
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                for _ in range(reps):
                    fn()
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(side)
            for _ in range(5):
                g.replay()
            e1.record(side)
            torch.cuda.synchronize()
            return round(e0.elapsed_time(e1) * 1e3 / (5 * reps), 2)
        except Exception:  # noqa: BLE001
            return None


def sweep_point(log_n, variant, log_r, rng, args, ref, out, fused_basis=None):
    n = 1 << log_n
    lib = nt._lib
    if log_n > COL_LOG_R:
        lib.call("nttmul_set_split", log_n, log_r)
        if log_n <= 16:  # the cluster schedule has its own fixed split
            lib.call("nttmul_set_schedule", 1, log_n, lib.SCHED_THREE)
    try:
        plan = nt.build_plan(n, bits=60, seed=0, variant=variant)
        red = plan.red_args  # (q, mode, mu, s_in, s_out)
        q = plan.q
        batch = max(1, min(args.batch, (1 << 27) // n))
        host = np.stack([rng.integers(0, q, n, dtype=np.uint64) for _ in range(2)])
        split = f"{1 << (log_n - log_r)}x{1 << log_r}"
        row = {"cfg": "cfg5", "log_n": log_n, "variant": variant, "split": split,
               "log_n2": log_r}
        if not args.ncu_plan:
            # parity: polynomial 0 of a 2-row batch vs the C oracle
            x = torch.from_numpy(host.copy()).cuda()
            nt.kernels.ntt_ct(x, plan.tw_fwd, *red, False, None)
            f, iv = oracle.twiddles(q, plan.psi, log_n)
            want = host[0].copy()
            oracle.ntt_ct(want, f, *plan.red_args, False)
            fwd_ok = np.array_equal(x[0].cpu().numpy(), want)
            nt.kernels.intt_gs(x, plan.tw_inv, q, (q + 1) // 2, *red[1:], True, False, None)
            inv_ok = np.array_equal(x.cpu().numpy(), host)
            row["parity"] = "bit-exact" if fwd_ok and inv_ok else "MISMATCH"
        one = torch.from_numpy(host[:1].copy()).cuda()
        many = torch.from_numpy(host[np.arange(batch) % 2].copy()).cuda()
        pairs_f, _ = nt.kernels._pairs_for(plan.tw_fwd, int(q))
        pairs_i, w1 = nt.kernels._pairs_for(plan.tw_inv, int(q))

        def c_ntt(t):
            return lambda: lib.call(
                "nttmul_ntt_ct", t.data_ptr(), pairs_f.data_ptr(), *(int(v) for v in red),
                0, log_n, t.shape[0], torch.cuda.current_stream().cuda_stream)

        def c_intt(t):
            return lambda: lib.call(
                "nttmul_intt_gs", t.data_ptr(), pairs_i.data_ptr(), int(q), (int(q) + 1) // 2,
                *(int(v) for v in red[1:]), 1, 0, log_n, t.shape[0], int(w1),
                torch.cuda.current_stream().cuda_stream)

        if args.ncu_plan:
            c_ntt(many)()
            torch.cuda.synchronize()
            row["ncu_launches"] = 2 if log_n > COL_LOG_R else 1
            row["batch"] = batch
            out.write(json.dumps(row) + "\n")
            out.flush()
            return
        row["ntt_device_us"] = graph_us(c_ntt(one))
        row["intt_scaled_device_us"] = graph_us(c_intt(one))
        row["ntt_api_us"] = round(1e3 * timed(
            lambda: nt.kernels.ntt_ct(one, plan.tw_fwd, *red, False, None), 50), 2)
        row["intt_scaled_api_us"] = round(1e3 * timed(
            lambda: nt.kernels.intt_gs(one, plan.tw_inv, q, (q + 1) // 2, *red[1:], True,
                                       False, None), 50), 2)
        ms = timed(c_ntt(many), 10)
        row["batch"] = batch
        row["ntt_batch_us_per_poly"] = round(1e3 * ms / batch, 3)
        row["ntt_gbfly_s"] = round(batch * (n // 2) * log_n / (ms / 1e3) / 1e9, 1)
        ms = timed(c_intt(many), 10)
        row["intt_batch_us_per_poly"] = round(1e3 * ms / batch, 3)
        if fused_basis is not None:  # the fused product at this split (8 limbs)
            L = fused_basis.num_limbs
            B = max(1, (1 << 27) // (n * L * 2))
            A = torch.from_numpy(np.stack([host[np.arange(L) % 2]] * B)).cuda()
            C, W = torch.empty_like(A), torch.empty_like(A)
            if log_n <= 16:
                lib.call("nttmul_set_schedule", 0, log_n, lib.SCHED_THREE)
            ms = timed(lambda: nt.polymul_rns_batch(A, A, fused_basis, out=C, workspace=W), 10)
            if log_n <= 16:
                lib.call("nttmul_set_schedule", 0, log_n, lib.SCHED_AUTO)
            mm = B * L * ((3 * n // 2) * (log_n - 1) + 2 * n)
            row["fused_ct_per_s"] = round(B / ms * 1e3, 1)
            row["fused_gmodmul_s"] = round(mm / ms / 1e6, 1)
            row["fused_batch"] = f"{B}x{L}"
        # data x data Barrett products of this variant (mulmod_loop, XOR sink;
        # one reduction per element per call - the pass count only sets the
        # parity of the XOR, like the reference's loop)
        a = torch.from_numpy(host[0].copy()).cuda()
        b = torch.from_numpy(host[1].copy()).cuda()
        ms = timed(lambda: nt.kernels.mulmod_loop(a, b, *red, 1), 20)
        row["mulmod_loop_gred_s"] = round(n / (ms / 1e3) / 1e9, 2)
        if ref is not None and log_r == splits(log_n)[0]:  # the reference CPU transform (1 core)
            rplan = ref.build_plan(n, bits=60, seed=0, variant=variant)
            assert rplan.q == q and rplan.psi == plan.psi
            best = 1e9
            for _ in range(3):
                p = ref.Polynomial(host[0].copy())
                t0 = time.perf_counter()
                ref.ntt_ct(p, rplan)
                best = min(best, time.perf_counter() - t0)
            row["ref_cpu_ntt_us"] = round(best * 1e6, 1)
        out.write(json.dumps(row) + "\n")
        out.flush()
    finally:
        if log_n > COL_LOG_R:
            lib.call("nttmul_set_split", log_n, 0)
            if log_n <= 16:
                lib.call("nttmul_set_schedule", 1, log_n, lib.SCHED_AUTO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--min-log", type=int, default=10)
    ap.add_argument("--max-log", type=int, default=17)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--ncu-plan", action="store_true")
    args = ap.parse_args()
    out = open(args.out, "w") if args.out else sys.stdout
    rng = np.random.default_rng(0)
    ref = None if args.ncu_plan else oracle.reference()
    for log_n in range(args.min_log, args.max_log + 1):
        fb = nt.RnsBasis.build(1 << log_n, 60, 8, seed=0) if log_n > COL_LOG_R else None
        if not args.ncu_plan:
            for variant in VARIANTS[:-1]:
                sweep_point(log_n, variant, splits(log_n)[0], rng, args, ref, out)
        for log_r in splits(log_n):
            sweep_point(log_n, "proposed", log_r, rng, args, ref, out,
                        None if args.ncu_plan else fb)


if __name__ == "__main__":
    main()
