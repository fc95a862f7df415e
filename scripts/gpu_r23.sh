cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=10 -k "crt or rns or naive" > gpurun_out/pytest_r23.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r23.log
