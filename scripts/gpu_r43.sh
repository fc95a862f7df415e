# final bench lines (both arms) + cfg5 sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r43.log 2>&1; echo "exit $?" >> gpurun_out/bench_r43.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r43.log 2>&1; echo "exit $?" >> gpurun_out/bench_ref_r43.log
timeout 900 python scripts/ntt_sweep.py --out gpurun_out/cfg5_sweep_r43.jsonl > gpurun_out/cfg5_r43.log 2>&1; echo "exit $?" >> gpurun_out/cfg5_r43.log
