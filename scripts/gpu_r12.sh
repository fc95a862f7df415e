# parity tests on the default library, then a variant sweep, then a full bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r12.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r12.log
VARIANTS="default carry nolazy" PIPES="0,0" TAG=r12 bash scripts/sweep.sh
timeout 600 python bench.py > gpurun_out/bench_r12.log 2>&1; echo "exit $?" >> gpurun_out/bench_r12.log
