# PM-shaped moduli (LB = 33): parity + bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_pm.log 2>&1; echo "exit $?" >> gpurun_out/pytest_pm.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_pm.log 2>&1; echo "exit $?" >> gpurun_out/bench_pm.log
