cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in e4m2 e3m1 e3m2; do
  NTTMUL_LIB=build/variants/lib_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_$v.log 2>&1; echo "exit $?" >> gpurun_out/pytest_$v.log
done
VARIANTS="e4m2 e3m1 e3m2" PIPES="0,1" TAG=r3 bash scripts/sweep.sh
