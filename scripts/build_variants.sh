#!/usr/bin/env bash
# Build experimental library variants into build/variants/ (for sweeps).
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
for spec in "$@"; do
  name="${spec%%:*}"; defs="${spec#*:}"
  flags=""
  for d in ${defs//,/ }; do flags="$flags -D$d"; done
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -Iinclude $flags -o build/variants/lib_$name.so paper_2209_01290_b200/csrc/capi.cu &
done
wait
ls -la build/variants
