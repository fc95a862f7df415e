cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/roof.py <<'PY'
import ctypes, torch, sys
sys.path.insert(0, '.')
import paper_2209_01290_b200 as nt
plan = nt.build_plan(1 << 16, bits=60, seed=0)
limb = plan.limb()
sink = torch.zeros(1, dtype=torch.uint64, device='cuda')
cnt = ctypes.c_double()
for kind in (2, 1, 0):
    nt._lib.call("nttmul_modmul_roof", ctypes.byref(limb), kind, 148 * 8, 256, 400, sink.data_ptr(), ctypes.byref(cnt), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none -k regex:modmul_roof -c 3 -o gpurun_out/prof_roof python /tmp/roof.py > gpurun_out/ncu_roof.log 2>&1
echo "exit $?" >> gpurun_out/ncu_roof.log
