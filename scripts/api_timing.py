"""Back-to-back standalone transforms through the Python API, timed with
CUDA events on the launching stream (what bench.py's ntt_us.api_us
reports): per call, 50 calls after 5 warm-ups, median of 7 repetitions,
for the default (grid) and the pass schedule.  Run once with and once
without NTTB_NO_GRAPH=1 to see the launch-graph cache's effect on the
device timeline.

    python scripts/api_timing.py; NTTB_NO_GRAPH=1 python scripts/api_timing.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_01290_b200 as nt  # noqa: E402

lib = nt._lib


def per_call_us(fn, calls=50, reps=7):
    """(events per call, host issue time per call), medians, in us."""
    import time
    stream = torch.cuda.current_stream()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    out, host = [], []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        for _ in range(calls):
            fn()
        host.append((time.perf_counter() - t0) * 1e6 / calls)
        e1.record(stream)
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3 / calls)
    return round(sorted(out)[reps // 2], 2), round(sorted(host)[reps // 2], 2)


def main():
    for log_n in (13, 16):
        n = 1 << log_n
        plan = nt.build_plan(n, bits=60, seed=0)
        x = torch.from_numpy(np.random.default_rng(0).integers(0, plan.q, n, dtype=np.uint64)).cuda()
        rec = {"log_n": log_n, "graph_cache": os.environ.get("NTTB_NO_GRAPH") is None}
        for sched, name in ((lib.SCHED_AUTO, "grid"), (lib.SCHED_PASSES, "passes")):
            lib.call("nttmul_set_schedule", 1, log_n, sched)
            rec[name + "_api_us"] = per_call_us(
                lambda: nt.kernels.ntt_ct(x, plan.tw_fwd, *plan.red_args, False, None))
        lib.call("nttmul_set_schedule", 1, log_n, lib.SCHED_AUTO)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
