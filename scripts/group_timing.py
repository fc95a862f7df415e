"""Group-kernel phase breakdown (steady-state product k=4) from a
NTTB_PHASE_TIMING build."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("NTTMUL_LIB", "build/variants/lib_phase.so")
import paper_2209_01290_b200 as nt
B, L = 16, 21
basis = nt.RnsBasis.build(1 << 16, 60, L, seed=0)
A = torch.zeros((B, L, 1 << 16), dtype=torch.uint64, device="cuda")
Bm = torch.zeros_like(A)
for _ in range(3):
    nt.polymul_rns_batch(A, Bm, basis)
torch.cuda.synchronize()
lib = nt._lib.load()
rows = 288
buf = (ctypes.c_ulonglong * (8 * 65536))()
assert lib.nttmul_debug_phases(buf, 65536) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(65536, 8)[:rows].astype(np.int64)
d = np.diff(t[:, :6], axis=1)
names = ["wait1 (all P1(k) done)", "P2 row pass + arrive", "P1(k+1) columns + arrive",
         "wait2 (all P2(k) done)", "P3 inverse columns"]
tot = d.sum(1).mean()
for i, n in enumerate(names):
    print(f"{n:32s} mean {d[:, i].mean():9.0f}  min {d[:, i].min():9.0f}  max {d[:, i].max():9.0f} cycles  {d[:, i].mean() / tot * 100:5.1f}%")
print(f"{'period':32s} {tot:9.0f} cycles")
