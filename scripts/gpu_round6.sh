cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in pf pfldg; do
NTTMUL_LIB=build/variants/lib_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_r6_$v.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r6_$v.log
done
VARIANTS="default pf ldg pfldg pfm1" PIPES="0,0" TAG=r6 bash scripts/sweep.sh
