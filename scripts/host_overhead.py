"""Host issue cost per call of a single standalone transform (n = 2^13 ..
2^17): wall time per call of back-to-back calls WITHOUT synchronising
(the host side only - the device queue absorbs the work), for the raw
C-ABI entry point through ctypes with pre-built arguments and for the
Python API (kernels.ntt_ct).  One JSON line per size.

    python scripts/host_overhead.py
"""
from __future__ import annotations

import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_01290_b200 as nt  # noqa: E402

lib = nt._lib


def per_call_us(fn, reps=100):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(5):
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        best = min(best, (time.perf_counter() - t0) / reps * 1e6)
        torch.cuda.synchronize()
    return round(best, 2)


def main():
    for log_n in range(13, 18):
        n = 1 << log_n
        plan = nt.build_plan(n, bits=60, seed=0)
        q, mode, mu, s_in, s_out = plan.red_args
        pf, _ = nt.kernels._pairs_for(plan.tw_fwd, q)
        x = torch.zeros((1, n), dtype=torch.uint64, device="cuda")
        fn = lib.load().nttmul_ntt_ct
        st = torch.cuda.current_stream().cuda_stream
        xp, pp = x.data_ptr(), pf.data_ptr()
        rec = {
            "log_n": log_n,
            "raw_ctypes_us": per_call_us(lambda: fn(xp, pp, q, mode, mu, s_in, s_out, 0, log_n,
                                                    1, st)),
            "lib_call_us": per_call_us(lambda: lib.call("nttmul_ntt_ct", xp, pp, q, mode, mu,
                                                        s_in, s_out, 0, log_n, 1, st)),
            "api_us": per_call_us(lambda: nt.kernels.ntt_ct(x, plan.tw_fwd, q, mode, mu, s_in,
                                                            s_out, False, None)),
            "torch_zero_us": per_call_us(lambda: x.zero_()),
        }
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
