"""Launch driver for ncu: three forward + inverse pairs of one standalone
transform of 2^LOG_N words under the default schedule, then under the grid
schedule (run with NTTB_NO_GRAPH=1 so every launch is a kernel, not a graph).

    NTTB_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none \
        python scripts/grid_ncu.py 16
"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_01290_b200 as nt
lib = nt._lib
log_n = int(sys.argv[1]); n = 1 << log_n
plan = nt.build_plan(n, bits=60, seed=0)
q, mode, mu, s_in, s_out = plan.red_args
pf, _ = nt.kernels._pairs_for(plan.tw_fwd, q)
pi, w1 = nt.kernels._pairs_for(plan.tw_inv, q)
x = torch.from_numpy(np.random.default_rng(1).integers(0, q, (1, n), dtype=np.uint64)).cuda()
for sched in (lib.SCHED_AUTO, lib.SCHED_GRID):
    lib.call("nttmul_set_schedule", 1, log_n, sched)
    for _ in range(3):
        lib.call("nttmul_ntt_ct", x.data_ptr(), pf.data_ptr(), q, mode, mu, s_in, s_out, 0, log_n, 1, 0)
        lib.call("nttmul_intt_gs", x.data_ptr(), pi.data_ptr(), q, (q + 1) // 2, mode, mu, s_in, s_out, 1, 0, log_n, 1, w1, 0)
torch.cuda.synchronize()
