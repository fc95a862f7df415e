cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=10 > gpurun_out/pytest_r30.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r30.log
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r30_$i.log 2>&1; done
