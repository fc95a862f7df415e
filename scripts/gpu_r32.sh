cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARIANTS="default p4 p6 s3 default p4" PIPES="0,0" TAG=r32 bash scripts/sweep.sh
