"""Row-kernel phase breakdown from a NTTB_PHASE_TIMING build (debug)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("NTTMUL_LIB", "build/variants/lib_phase.so")
import paper_2209_01290_b200 as nt
B, L = 8, 21
basis = nt.RnsBasis.build(1 << 16, 60, L, seed=0)
A = torch.zeros((B, L, 1 << 16), dtype=torch.uint64, device="cuda")
Bm = torch.zeros_like(A)
for _ in range(3):
    nt.polymul_rns_batch(A, Bm, basis)
torch.cuda.synchronize()
lib = nt._lib.load()
rows = min(B * L * 16, 1 << 16)
buf = (ctypes.c_ulonglong * (8 * rows))()
assert lib.nttmul_debug_phases(buf, rows) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(rows, 8).astype(np.int64)
d = np.diff(t[:, :5], axis=1)
names = ["pass0 (global load + 3 stages, a,b)", "head passes 1-2 (a,b)", "tail (fwd+middle+inv)",
         "inverse head passes + store"]
tot = d.sum(1).mean()
for i, n in enumerate(names):
    print(f"{n:40s} {d[:, i].mean():9.0f} cycles  {d[:, i].mean() / tot * 100:5.1f}%")
print(f"{'total per CTA':40s} {tot:9.0f} cycles")
