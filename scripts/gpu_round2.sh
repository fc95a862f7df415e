cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
VARIANTS="m1 m2 m3" PIPES="0,1 1,3 2,3 4,2 2,4" TAG=r2 bash scripts/sweep.sh
