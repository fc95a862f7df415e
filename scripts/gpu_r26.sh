cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARIANTS="default colvec1 colminb3 colminb4 colvec1m4 colvec1m3" PIPES="0,0" TAG=r26 bash scripts/sweep.sh
