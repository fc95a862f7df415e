# ncu --set full of one kernel matched by $KREGEX (default: fused row kernel)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"${KREGEX:-row_kernel}" -c ${COUNT:-1} -o gpurun_out/prof_${TAG:-x} \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --batch 8 ${EXTRA} > gpurun_out/ncu_${TAG:-x}.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_${TAG:-x}.log
