cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r11.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r11.log
VARIANTS="default" PIPES="0,0" TAG=r11 bash scripts/sweep.sh
