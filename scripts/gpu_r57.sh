cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r57.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r57.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_r57_$i.log 2>&1; done
timeout 600 python bench.py --log-n 17 --limbs 32 --batch 8 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4_r57.log 2>&1
