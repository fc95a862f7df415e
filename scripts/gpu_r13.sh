cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r13.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r13.log
timeout 300 python scripts/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_r13.log 2>&1; echo "exit $?" >> gpurun_out/bench_r13.log
timeout 900 ncu --set full --section InstructionStats --section WarpStateStats --clock-control none --import-source on \
  -k regex:"row_kernel" -c 1 -o gpurun_out/prof_r13 \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --batch 8 > gpurun_out/ncu_r13.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_r13.log
