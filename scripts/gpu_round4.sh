cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_r4.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r4.log
VARIANTS="default e4m2" PIPES="0,0 1,0 2,0 3,0 4,0" TAG=r4 bash scripts/sweep.sh
