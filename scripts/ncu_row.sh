# One ncu --set full capture of the fused row kernel (and the column kernels)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"row_kernel|col_kernel" -c 3 -o gpurun_out/prof_${TAG:-r1} \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --batch 8 > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full.log
