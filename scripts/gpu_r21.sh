cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NTTMUL_LIB=build/variants/lib_phase.so timeout 300 python scripts/group_timing.py > gpurun_out/group_timing.txt 2>&1
