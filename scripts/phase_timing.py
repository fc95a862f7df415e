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
order = [0, 5, 1, 6, 2, 3, 4]
names = ["a pass0 (global load + 3 stages)", "wait b (cp.async) + barrier", "b pass0 (smem)",
         "passes 1-2 (a, b)", "tail (fwd + middle + inv)", "inverse passes + store"]
d = np.diff(t[:, order], axis=1)
tot = d.sum(1).mean()
for i, n in enumerate(names):
    print(f"{n:40s} {d[:, i].mean():9.0f} cycles  {d[:, i].mean() / tot * 100:5.1f}%")
print(f"{'total (warp 0)':40s} {tot:9.0f} cycles")
print(f"{'CTA lifetime (start -> last warp done)':40s} {(t[:, 7] - t[:, 0]).mean():9.0f} cycles")
sm_start = t[:, 0]
print("rows", rows, "span of all CTAs (cycles, per-SM clocks differ)", int(t[:, 7].max() - t[:, 0].min()))
