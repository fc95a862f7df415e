"""One-launch grid schedule (NTTMUL_SCHED_GRID, csrc/grid_kernels.cuh) vs
the previous default latency schedule for a single standalone ntt_ct /
intt_gs (scaled) of n = 2^13 .. 2^17: device time per call from CUDA graphs
of back-to-back C-ABI calls (9 interleaved repetitions after a clock warm-up;
min and median), each grid result checked bit-for-bit against the other
schedule.  The grid geometry (2^A rows, 2^LOG_E elements per thread) comes
from NTTB_GRID_A / NTTB_GRID_E, which only a library built with
-DNTTB_GRID_SWEEP honours:

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \
        -shared -DNTTB_GRID_SWEEP -I include -o build/libnttmul_sweep.so \
        paper_2209_01290_b200/csrc/capi.cu
    for e in 1 2 3; do for a in 5 6 7 8; do NTTMUL_LIB=build/libnttmul_sweep.so \
        NTTB_GRID_E=$e NTTB_GRID_A=$a python scripts/grid_sweep.py; done; done

With the default library (no variables) it compares the built-in geometry
with NTTMUL_SCHED_PASSES.  One JSON line per point.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_01290_b200 as nt  # noqa: E402

lib = nt._lib
REPS = 9
CALLS = 20


def graph_fn(fn):
    """A CUDA graph of CALLS back-to-back calls of fn on a side stream."""
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for _ in range(CALLS):
                fn()
    torch.cuda.synchronize()
    return g


def replay_us(g, replays=10):
    stream = torch.cuda.current_stream()
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(replays):
        g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) * 1e3 / (replays * CALLS), 2)


def warm(g, seconds=0.3):
    """Replay for a while so the clocks ramp before the timed repetitions."""
    import time
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        for _ in range(20):
            g.replay()
        torch.cuda.synchronize()
VALID = {13: (5, 6), 14: (6, 7), 15: (6, 7), 16: (7, 8), 17: (7, 8)}


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, nargs="+", default=[1],
                    help="polynomials per call (the grid launch holds batch x 2^A CTAs)")
    args = ap.parse_args()
    a_env = int(os.environ.get("NTTB_GRID_A", "0"))
    for log_n, batch in [(ln, b) for b in args.batch for ln in range(13, 18)]:
        if a_env and a_env not in VALID[log_n]:  # (sweep library only)
            continue
        n = 1 << log_n
        plan = nt.build_plan(n, bits=60, seed=0)
        q, mode, mu, s_in, s_out = plan.red_args
        pf, _ = nt.kernels._pairs_for(plan.tw_fwd, q)
        pi, w1 = nt.kernels._pairs_for(plan.tw_inv, q)
        src = torch.from_numpy(np.random.default_rng(log_n).integers(
            0, q, (batch, n), dtype=np.uint64)).cuda()
        x = torch.empty_like(src)
        rec = {"log_n": log_n, "batch": batch, "grid_a": a_env,
               "grid_e": int(os.environ.get("NTTB_GRID_E", "0"))}
        outs, fns = {}, {}
        base = lib.SCHED_PASSES if batch == 1 else lib.SCHED_AUTO  # (auto: column / row)
        for sched, name in ((base, "default"), (lib.SCHED_GRID, "grid")):
            lib.call("nttmul_set_schedule", 1, log_n, sched)

            def fwd():
                lib.call("nttmul_ntt_ct", x.data_ptr(), pf.data_ptr(), q, mode, mu, s_in, s_out, 0,
                         log_n, batch, torch.cuda.current_stream().cuda_stream)

            def inv():
                lib.call("nttmul_intt_gs", x.data_ptr(), pi.data_ptr(), q, (q + 1) // 2, mode, mu,
                         s_in, s_out, 1, 0, log_n, batch, w1, torch.cuda.current_stream().cuda_stream)

            x.copy_(src)
            base = x.clone()
            fwd()
            y = x.clone()
            inv()
            outs[name] = (y.cpu(), x.cpu(), base.cpu())
            # graphs bind the launches of this schedule
            fns[name] = (graph_fn(fwd), graph_fn(inv))
        warm(fns["grid"][0])
        for name, (gf, gi) in fns.items():
            rec[name + "_ntt_us"] = []
            rec[name + "_intt_us"] = []
        for _ in range(REPS):  # interleaved repetitions (clock drift hits both)
            for name, (gf, gi) in fns.items():
                rec[name + "_ntt_us"].append(replay_us(gf))
                rec[name + "_intt_us"].append(replay_us(gi))
        for k in [k for k in rec if k.endswith("_us")]:
            v = sorted(rec[k])
            rec[k] = {"min": v[0], "median": v[len(v) // 2]}
        lib.call("nttmul_set_schedule", 1, log_n, lib.SCHED_AUTO)
        rec["bit_exact"] = bool(torch.equal(outs["grid"][0], outs["default"][0]) and
                                torch.equal(outs["grid"][1], outs["default"][1]) and
                                torch.equal(outs["grid"][1], outs["grid"][2]))
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
