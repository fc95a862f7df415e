cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r44.log 2>&1; echo "exit $?" >> gpurun_out/bench_r44.log
timeout 900 python scripts/ntt_sweep.py --out gpurun_out/cfg5_sweep_r44.jsonl > gpurun_out/cfg5_r44.log 2>&1; echo "exit $?" >> gpurun_out/cfg5_r44.log
