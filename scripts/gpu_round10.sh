cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_r10.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r10.log
VARIANTS="default nopb pbe4" PIPES="0,0" TAG=r10 bash scripts/sweep.sh
