cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=10 > gpurun_out/pytest_r34.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r34.log
VARIANTS="default nofast default nofast" PIPES="0,0" TAG=r34 bash scripts/sweep.sh
