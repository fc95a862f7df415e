cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARIANTS="default twpf minb1 e4" PIPES="0,0" TAG=r18 bash scripts/sweep.sh
./scripts/microbench/pipes2 > gpurun_out/pipes2.txt 2>&1
