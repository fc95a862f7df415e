cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=10 > gpurun_out/pytest_r29.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r29.log
VARIANTS="default nopersist default nopersist" PIPES="0,0" TAG=r29 bash scripts/sweep.sh
