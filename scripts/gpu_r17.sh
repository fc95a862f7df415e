cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r17.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r17.log
VARIANTS="default nopf colpipe" PIPES="0,0" TAG=r17 bash scripts/sweep.sh
NTTMUL_LIB=build/variants/lib_phase.so timeout 300 python scripts/phase_timing.py > gpurun_out/phase_r17.txt 2>&1
