"""Single-transform latency of the standalone ntt_ct / intt_gs (scaled) per
schedule: the default (column kernel + row kernel, per-size split) vs the
latency schedule (strided passes of <= 3 column stages + 1024-word rows,
NTTMUL_SCHED_PASSES), batch 1 and 4.  Device time per call from a CUDA
graph of back-to-back C-ABI launches (no host overhead) and through the
Python API.  One JSON line per point.

    python scripts/latency_sweep.py [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_01290_b200 as nt  # noqa: E402
from ntt_sweep import graph_us, timed  # noqa: E402

lib = nt._lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    out = open(args.out, "w") if args.out else sys.stdout
    for log_n in range(13, 18):
        n = 1 << log_n
        plan = nt.build_plan(n, bits=60, seed=0)
        q, mode, mu, s_in, s_out = plan.red_args
        pf, _ = nt.kernels._pairs_for(plan.tw_fwd, q)
        pi, w1 = nt.kernels._pairs_for(plan.tw_inv, q)
        for batch in (1, 4):
            x = torch.zeros((batch, n), dtype=torch.uint64, device="cuda")
            for sched, name in ((lib.SCHED_AUTO, "default"), (lib.SCHED_PASSES, "passes")):
                lib.call("nttmul_set_schedule", 1, log_n, sched)

                def fwd():
                    lib.call("nttmul_ntt_ct", x.data_ptr(), pf.data_ptr(), q, mode, mu, s_in,
                             s_out, 0, log_n, batch, torch.cuda.current_stream().cuda_stream)

                def inv():
                    lib.call("nttmul_intt_gs", x.data_ptr(), pi.data_ptr(), q, (q + 1) // 2, mode,
                             mu, s_in, s_out, 1, 0, log_n, batch, w1,
                             torch.cuda.current_stream().cuda_stream)

                rec = {"log_n": log_n, "batch": batch, "schedule": name,
                       "ntt_device_us": graph_us(fwd), "intt_device_us": graph_us(inv),
                       "ntt_api_us": round(1e3 * timed(
                           lambda: nt.kernels.ntt_ct(x, plan.tw_fwd, q, mode, mu, s_in, s_out,
                                                     False, None), 50), 2)}
                out.write(json.dumps(rec) + "\n")
                out.flush()
            lib.call("nttmul_set_schedule", 1, log_n, lib.SCHED_AUTO)


if __name__ == "__main__":
    main()
