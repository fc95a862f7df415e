#!/usr/bin/env bash
# Sweep library variants x pipeline settings with short bench runs.
# usage: VARIANTS="m1 m2" PIPES="0,1 2,3" bash scripts/sweep.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/sweep_${TAG:-x}.jsonl
: > $out
for v in ${VARIANTS:-default}; do
  lib=""
  [ "$v" != "default" ] && lib="build/variants/lib_$v.so"
  for p in ${PIPES:-0,1}; do
    res=$(NTTMUL_LIB=$lib timeout 300 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e --pipeline $p ${EXTRA} 2>&1 | tail -1)
    echo "{\"variant\": \"$v\", \"pipe\": \"$p\", \"res\": $res}" >> $out 2>/dev/null || echo "$v $p FAILED: $res" >> $out
  done
done
