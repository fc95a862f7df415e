cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r20.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r20.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r20.log 2>&1; echo "exit $?" >> gpurun_out/bench_r20.log
