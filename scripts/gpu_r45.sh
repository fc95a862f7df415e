# supplementary bench lines: cfg2 (N=2^14, 8 limbs, 64 ct) and cfg4 (N=2^17, 32 limbs, 8 ct)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --log-n 14 --limbs 8 --batch 64 --cpu-seconds 5 > gpurun_out/bench_cfg2_r45.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg2_r45.log
timeout 600 python bench.py --log-n 17 --limbs 32 --batch 8 --cpu-seconds 5 > gpurun_out/bench_cfg4_r45.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg4_r45.log
