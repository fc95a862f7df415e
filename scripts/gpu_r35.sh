cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARIANTS="default midonly nolb32 default midonly" PIPES="0,0" TAG=r35 bash scripts/sweep.sh
