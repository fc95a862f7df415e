# occupancy experiments on the fused row kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/occ_r40.txt; : > $out
NTTB_DEBUG_OCC=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e >> $out 2>&1
NTTB_DEBUG_OCC=1 NTTB_ROW_EXTRA_SMEM=57344 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e >> $out 2>&1
NTTB_DEBUG_OCC=1 timeout 300 python scripts/phase_timing.py >> $out 2>&1
NTTB_DEBUG_OCC=1 NTTB_ROW_EXTRA_SMEM=57344 timeout 300 python scripts/phase_timing.py >> $out 2>&1
