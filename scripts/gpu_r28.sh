cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"row_kernel|col_kernel" -c 3 -o gpurun_out/prof_r28 \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --batch 8 > gpurun_out/ncu_r28.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_r28.log
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r28.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_r28.log 2>&1
