cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARIANTS="default s3 tc128s4 plain" PIPES="0,0" TAG=r16 bash scripts/sweep.sh
