"""Launch driver for ncu: three forward + inverse pairs of one standalone
transform of 2^LOG_N words under the pass schedule, then under the grid
schedule, then three single fused limb-products (one-launch grid_fused
kernel).  Run with NTTB_NO_GRAPH=1 so every launch is a kernel, not a graph:

    NTTB_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none \\
        python scripts/grid_ncu.py 16
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_01290_b200 as nt  # noqa: E402

lib = nt._lib
log_n = int(sys.argv[1])
n = 1 << log_n
plan = nt.build_plan(n, bits=60, seed=0)
q, mode, mu, s_in, s_out = plan.red_args
pf, _ = nt.kernels._pairs_for(plan.tw_fwd, q)
pi, w1 = nt.kernels._pairs_for(plan.tw_inv, q)
x = torch.from_numpy(np.random.default_rng(1).integers(0, q, (1, n), dtype=np.uint64)).cuda()
for sched in (lib.SCHED_PASSES, lib.SCHED_GRID):
    lib.call("nttmul_set_schedule", 1, log_n, sched)
    for _ in range(3):
        lib.call("nttmul_ntt_ct", x.data_ptr(), pf.data_ptr(), q, mode, mu, s_in, s_out, 0,
                 log_n, 1, 0)
        lib.call("nttmul_intt_gs", x.data_ptr(), pi.data_ptr(), q, (q + 1) // 2, mode, mu,
                 s_in, s_out, 1, 0, log_n, 1, w1, 0)
lib.call("nttmul_set_schedule", 1, log_n, lib.SCHED_AUTO)
fused = nt.FusedPlan.from_plan(plan)
a = x[0].clone()
for _ in range(3):
    nt.polymul_fused(a, a, fused)
torch.cuda.synchronize()
