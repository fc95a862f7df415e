cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r37.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r37.log
VARIANTS="default notw c4 c4i8 default notw" PIPES="0,0" TAG=r37 STEPS=20 bash scripts/sweep.sh
