# row kernel at 1 CTA/SM (smem padding) so the column kernels of the other
# half co-reside, x split parts
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/sweep_r41.jsonl; : > $out
for v in default p4 p6 s3p6; do
  lib=""; [ "$v" != "default" ] && lib="build/variants/lib_$v.so"
  for pad in 0 57344 40960; do
    res=$(NTTMUL_LIB=$lib NTTB_ROW_EXTRA_SMEM=$pad timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1)
    echo "{\"variant\": \"$v\", \"pad\": $pad, \"res\": $res}" >> $out
  done
done
