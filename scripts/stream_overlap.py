"""Does splitting the cfg3 batch over 2-4 CUDA streams (so the HBM-bound
column kernels of one part overlap the integer-bound row kernel of another)
beat one launch sequence?  Prints ct/s per configuration."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2209_01290_b200 as nt  # noqa: E402

B, L, n = 16, 21, 1 << 16
basis = nt.RnsBasis.build(n, 60, L, seed=0)
q = torch.tensor(np.array(basis.primes, dtype=np.uint64).astype(np.int64), device="cuda").view(1, L, 1)
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.randint(0, 2**62, (B, L, n), dtype=torch.int64, device="cuda", generator=g) % q).to(torch.uint64)
Bm = (torch.randint(0, 2**62, (B, L, n), dtype=torch.int64, device="cuda", generator=g) % q).to(torch.uint64)
C = torch.empty_like(A)
W = torch.empty_like(A)
ref = nt.polymul_rns_batch(A, Bm, basis)
out = {}
for parts in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    step = B // parts

    def run():
        cur = torch.cuda.current_stream()
        for i, s in enumerate(streams):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                sl = slice(i * step, (i + 1) * step)
                nt.polymul_rns_batch(A[sl], Bm[sl], basis, out=C[sl], workspace=W[sl])
        for s in streams:
            cur.wait_stream(s)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    assert torch.equal(C, ref)
    out[f"streams{parts}"] = round(B * 10 / (e0.elapsed_time(e1) / 1e3), 1)
print(json.dumps(out))
