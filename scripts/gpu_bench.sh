cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_${TAG:-b}.log 2>&1; echo "exit $?" >> gpurun_out/pytest_${TAG:-b}.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_${TAG:-b}.json 2> gpurun_out/bench_${TAG:-b}.err; echo "exit $?" >> gpurun_out/bench_${TAG:-b}.err
