cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r24.log 2>&1; echo "exit $?" >> gpurun_out/bench_r24.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"crt_" -c 2 -o gpurun_out/prof_crt \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --batch 2 > gpurun_out/ncu_crt.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_crt.log
