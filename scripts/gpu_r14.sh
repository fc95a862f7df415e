cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r15.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r15.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r15.log 2>&1; echo "exit $?" >> gpurun_out/bench_r15.log
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"col_pipe" -c 2 -o gpurun_out/prof_r15 \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --batch 8 > gpurun_out/ncu_r15.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_r15.log
