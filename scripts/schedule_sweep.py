"""Three-launch vs cluster schedule (nttmul_set_schedule) for the fused RNS
product and the standalone transforms, device-timed with CUDA events.

    python scripts/schedule_sweep.py [--out file.jsonl]

One JSON line per (kind, log_n, schedule): ms per call, ct-polymul/s (fused)
or us per transform (standalone), Gmodmul/s of the reference op count."""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_01290_b200 as nt  # noqa: E402

lib = nt._lib
CFG = {13: (8, 64), 14: (8, 64), 15: (16, 16), 16: (21, 16)}  # log_n -> (limbs, batch)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    out = open(args.out, "w") if args.out else None
    for log_n, (L, B) in CFG.items():
        n = 1 << log_n
        basis = nt.RnsBasis.build(n, 60, L, seed=0)
        g = torch.Generator(device="cuda").manual_seed(log_n)
        q = torch.tensor(basis.primes, dtype=torch.float64, device="cuda")[None, :, None]
        A = (torch.rand((B, L, n), generator=g, device="cuda", dtype=torch.float64) * q
             ).to(torch.int64).to(torch.uint64)
        Bm = (torch.rand((B, L, n), generator=g, device="cuda", dtype=torch.float64) * q
              ).to(torch.int64).to(torch.uint64)
        C, W = torch.empty_like(A), torch.empty_like(A)
        res = {}
        for sched in (lib.SCHED_THREE, lib.SCHED_CLUSTER):
            lib.call("nttmul_set_schedule", 0, log_n, sched)
            ms = timed(lambda: nt.polymul_rns_batch(A, Bm, basis, out=C, workspace=W))
            res[sched] = C.clone()
            mm = B * L * ((3 * n // 2) * (log_n - 1) + 2 * n)
            rec = {"kind": "fused", "log_n": log_n, "limbs": L, "batch": B,
                   "schedule": "cluster" if sched == lib.SCHED_CLUSTER else "three",
                   "ms": round(ms, 4), "ct_per_s": round(B / ms * 1e3, 1),
                   "gmodmul_s": round(mm / ms / 1e6, 1)}
            print(json.dumps(rec), flush=True)
            if out:
                out.write(json.dumps(rec) + "\n")
        lib.call("nttmul_set_schedule", 0, log_n, lib.SCHED_AUTO)
        assert torch.equal(res[lib.SCHED_THREE], res[lib.SCHED_CLUSTER])
        plan = basis.plans[0]
        for batch in (1, 128):
            x = A[:, 0].reshape(-1, n)[:1].repeat(batch, 1).contiguous()
            for sched in (lib.SCHED_THREE, lib.SCHED_CLUSTER):
                lib.call("nttmul_set_schedule", 1, log_n, sched)
                pairs, _ = nt.kernels._pairs_for(plan.tw_fwd, plan.q)
                qq, mode, mu, s_in, s_out = plan.red_args
                st = torch.cuda.current_stream().cuda_stream

                def launch():
                    lib.call("nttmul_ntt_ct", x.data_ptr(), pairs.data_ptr(), qq, mode, mu,
                             s_in, s_out, 0, log_n, batch, st)

                ms = timed(launch, 50)
                rec = {"kind": "ntt_ct", "log_n": log_n, "batch": batch,
                       "schedule": "cluster" if sched == lib.SCHED_CLUSTER else "three",
                       "us_per_call": round(ms * 1e3, 2),
                       "us_per_transform": round(ms * 1e3 / batch, 3)}
                print(json.dumps(rec), flush=True)
                if out:
                    out.write(json.dumps(rec) + "\n")
            lib.call("nttmul_set_schedule", 1, log_n, lib.SCHED_AUTO)


if __name__ == "__main__":
    main()
