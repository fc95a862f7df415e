cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=10 --durations=8 > gpurun_out/pytest_r25.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r25.log
