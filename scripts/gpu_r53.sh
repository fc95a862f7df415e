# staggered split parts (part p's forward columns after part p-1's) x parts
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "cfg3 or full or batch" > gpurun_out/pytest_r53.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r53.log
VARIANTS="default nostag st3 st4 default nostag" PIPES="0,0" TAG=r53 STEPS=20 bash scripts/sweep.sh
