"""One-launch fused product (grid_fused_kernel, NTTMUL_SCHED_GRID for the
fused product) vs the three-launch column / row / column schedule, for a
few limb-products per call (n = 2^13 .. 2^17, 60-bit proposed-variant RNS
bases): device time per call from CUDA graphs of back-to-back C-ABI calls,
9 interleaved repetitions after a clock warm-up (min / median).  A forced
grid launch that does not fit co-resident is reported as null.  Each grid
result is checked bit-for-bit against the three-launch one.

    python scripts/grid_fused_sweep.py [--products 1 2 4]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_01290_b200 as nt  # noqa: E402
from grid_sweep import REPS, graph_fn, replay_us, warm  # noqa: E402

lib = nt._lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--products", type=int, nargs="+", default=[1, 2, 4])
    ap.add_argument("--bits", type=int, default=60)
    args = ap.parse_args()
    for log_n in range(13, 18):
        n = 1 << log_n
        for L in args.products:
            basis = nt.RnsBasis.build(n, args.bits, L, seed=0)
            fwd, inv, limbs = basis.device_tables()
            rng = np.random.default_rng(log_n)
            A = torch.from_numpy(np.stack([rng.integers(0, q, n, dtype=np.uint64)
                                           for q in basis.primes])[None]).cuda()
            B = torch.from_numpy(np.stack([rng.integers(0, q, n, dtype=np.uint64)
                                           for q in basis.primes])[None]).cuda()
            C = torch.empty_like(A)
            ws = torch.empty_like(A)
            mode = basis.mode

            def call():
                lib.call("nttmul_polymul_fused_rns", C.data_ptr(), A.data_ptr(), B.data_ptr(),
                         limbs.data_ptr(), fwd.data_ptr(), inv.data_ptr(), log_n, L, 1, mode,
                         ws.data_ptr(), torch.cuda.current_stream().cuda_stream)

            rec = {"log_n": log_n, "products": L}
            outs, graphs = {}, {}
            for sched, name in ((lib.SCHED_THREE, "three"), (lib.SCHED_GRID, "grid")):
                lib.call("nttmul_set_schedule", 0, log_n, sched)
                try:
                    call()
                except lib.NttmulError as exc:
                    rec[name + "_error"] = str(exc)[-80:]
                    continue
                torch.cuda.synchronize()
                outs[name] = C.clone()
                graphs[name] = graph_fn(call)
            lib.call("nttmul_set_schedule", 0, log_n, lib.SCHED_AUTO)
            warm(next(iter(graphs.values())))
            times = {k: [] for k in graphs}
            for _ in range(REPS):
                for k, g in graphs.items():
                    times[k].append(replay_us(g))
            for k, v in times.items():
                v.sort()
                rec[k + "_us"] = {"min": v[0], "median": v[len(v) // 2]}
            if len(outs) == 2:
                rec["bit_exact"] = bool(torch.equal(outs["three"], outs["grid"]))
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
