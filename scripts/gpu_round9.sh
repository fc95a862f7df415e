cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in p8m2 p16m2; do
NTTMUL_LIB=build/variants/lib_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_r9_$v.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r9_$v.log
done
VARIANTS="np p8m2 p8m1 p16m2 p16m1" PIPES="0,0" TAG=r9 bash scripts/sweep.sh
