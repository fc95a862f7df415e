cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_r8.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r8.log
NTTMUL_LIB=build/variants/lib_r11.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_r8_r11.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r8_r11.log
VARIANTS="default v1 v2m3 r11 r11v1" PIPES="0,0" TAG=r8 bash scripts/sweep.sh
