cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARIANTS="default f3 f4 f3i4 default f3 f4 f3i4" PIPES="0,0" TAG=r60 STEPS=20 bash scripts/sweep.sh
