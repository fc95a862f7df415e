cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r55.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r55.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_r55_$i.log 2>&1; done
