"""PCIe probe for the e2e path: raw pinned H2D / D2H / concurrent bandwidth
and polymul_rns_batch(host) at several chunk sizes (cfg3, 16 ciphertexts)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2209_01290_b200 as nt  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {}
nbytes = 352 << 20
h = torch.empty(nbytes // 8, dtype=torch.uint64, pin_memory=True)
d = torch.empty_like(h, device="cuda")
out["h2d_gbs"] = nbytes / timed(lambda: d.copy_(h, non_blocking=True)) / 1e6
out["d2h_gbs"] = nbytes / timed(lambda: h.copy_(d, non_blocking=True)) / 1e6
s2 = torch.cuda.Stream()
h2 = torch.empty_like(h, pin_memory=True)
d2 = torch.empty_like(d)


def both():
    d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


out["duplex_gbs_each"] = nbytes / timed(both) / 1e6
basis = nt.RnsBasis.build(1 << 16, 60, 21, seed=0)
rng = np.random.default_rng(0)
A = np.stack([np.stack([rng.integers(0, q, 1 << 16, dtype=np.uint64) for q in basis.primes])
              for _ in range(16)])
Ap = torch.from_numpy(A).pin_memory()
Bp = torch.from_numpy(A[::-1].copy()).pin_memory()
Cp = torch.empty_like(Ap).pin_memory()
per_ct = 21 * 8 << 16
for cts in (1, 2, 4, 8):
    nt.rns.HOST_CHUNK_BYTES = cts * per_ct
    ms = timed(lambda: nt.polymul_rns_batch(Ap, Bp, basis, out=Cp), reps=3)
    out[f"e2e_ct_s_chunk{cts}"] = 16 / (ms / 1e3)
print(json.dumps({k: round(v, 1) for k, v in out.items()}))
