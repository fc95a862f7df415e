cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r5.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r5.log
VARIANTS="default e4m2 e3m1" PIPES="0,0 2,0" TAG=r5 bash scripts/sweep.sh
