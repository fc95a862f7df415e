cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r46.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r46.log
timeout 600 python bench.py --log-n 17 --limbs 32 --batch 8 --no-cpu-baseline > gpurun_out/bench_cfg4_r46.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg4_r46.log
timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_r46.log 2>&1; echo "exit $?" >> gpurun_out/bench_r46.log
timeout 600 python scripts/ntt_sweep.py --min-log 17 --max-log 17 --out gpurun_out/cfg5_17_r46.jsonl > gpurun_out/cfg5_r46.log 2>&1
