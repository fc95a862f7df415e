"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    ./oracle/build_ref.sh            # builds the reference into oracle/_ref
    python tests/golden/make_golden.py

Everything here is computed by the reference package itself (nttmul with its
native Cython backend, imported from oracle/_ref) - these fixtures pin both
the C oracle (tests/test_oracle.py) and the GPU kernels (tests/test_gpu_*.py).
Inputs are reproducible from numpy's default_rng(seed); large outputs are
stored as SHA-256 digests of their little-endian uint64 bytes.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

nt = oracle.reference()
if nt is None:
    raise SystemExit("oracle/_ref missing: run ./oracle/build_ref.sh first")
from nttmul import backend  # noqa: E402

assert backend.active() == "native"


def rand(q: int, n: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, q, size=n, dtype=np.uint64)


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def counts_of(ctr) -> list[int]:
    return [ctr.modmul, ctr.modadd_sub, ctr.half_scalings, ctr.twiddle_loads, ctr.negations]


def plan_record(plan, bits=None, seed=None):
    return {
        "n": plan.n, "bits": bits, "seed": seed, "variant": plan.reduction_variant,
        "q": plan.q, "psi": plan.psi, "psi_inv": plan.psi_inv, "omega": plan.omega,
        "n_inv": plan.n_inv, "tw_fwd_sha": digest(plan.tw_fwd),
        "tw_inv_sha": digest(plan.tw_inv),
        "tw_fwd_head": [int(x) for x in plan.tw_fwd[:8]],
        "tw_inv_head": [int(x) for x in plan.tw_inv[:8]],
    }


def main():
    out = {"generator": "tests/golden/make_golden.py", "reference": "nttmul "
           + nt.__version__ + " (native backend, oracle/_ref)"}

    # ---- plans: prime / psi / twiddle tables (params.py:61-181) ----------
    plans = []
    grid = [(2, 10), (4, 12), (8, 14), (16, 20), (32, 28), (64, 28), (256, 30),
            (512, 62), (1024, 30), (4096, 60), (1 << 13, 60), (1 << 14, 60),
            (1 << 16, 60), (1 << 17, 60), (1 << 10, 62), (1 << 12, 28)]
    for n, bits in grid:
        for seed in (0, 1):
            plans.append(plan_record(nt.build_plan(n, bits=bits, seed=seed), bits, seed))
    for variant in ("builtin", "classical", "dhem"):
        plans.append(plan_record(nt.build_plan(256, bits=30, seed=0, variant=variant), 30, 0))
    out["plans"] = plans

    # ---- RNS bases (rns.py:44-58) - BASELINE configs -------------------------
    bases = []
    for n, bits, k in [(1 << 12, 60, 1), (1 << 14, 60, 8), (1 << 16, 60, 21),
                       (1 << 17, 60, 32), (64, 30, 4), (8, 30, 2)]:
        basis = nt.RnsBasis.build(n, bits, k, seed=0)
        bases.append({"n": n, "bits": bits, "k": k, "seed": 0,
                      "primes": list(basis.primes),
                      "psis": [p.psi for p in basis.plans],
                      "big_q": str(basis.big_q)})
    out["bases"] = bases

    # ---- full small vectors through the reference public API --------------
    vec = {}
    cases = []
    for n, bits in [(2, 10), (4, 12), (8, 14), (16, 20), (64, 28), (256, 30),
                    (512, 62), (1024, 60), (1024, 62), (2048, 30), (4096, 60)]:
        plan = nt.build_plan(n, bits=bits, seed=0)
        key = f"n{n}_b{bits}"
        a = rand(plan.q, n, 1000 + n)
        b = rand(plan.q, n, 2000 + n)
        x = rand(plan.q, n, 3000 + n)
        rec = {"key": key, "n": n, "bits": bits, "q": plan.q, "psi": plan.psi}
        vec[key + "_a"], vec[key + "_b"], vec[key + "_x"] = a, b, x

        c = nt.OpCounter()
        p = nt.Polynomial(a.copy())
        nt.ntt_ct(p, plan, c)
        vec[key + "_ntt"] = p.coeffs.copy()
        rec["ntt_counts"] = counts_of(c)

        c = nt.OpCounter()
        p = nt.Polynomial(x.copy(), "bit_reversed")
        nt.intt_gs(p, plan, c)
        vec[key + "_intt"] = p.coeffs.copy()
        rec["intt_counts"] = counts_of(c)

        c = nt.OpCounter()
        p = nt.Polynomial(x.copy(), "bit_reversed")
        nt.intt_gs_scaled(p, plan, c)
        vec[key + "_intts"] = p.coeffs.copy()
        rec["intts_counts"] = counts_of(c)

        if n >= 4:
            c = nt.OpCounter()
            p = nt.Polynomial(a.copy())
            nt.ntt_ct_truncated(p, plan, c)
            vec[key + "_nttt"] = p.coeffs.copy()
            rec["nttt_counts"] = counts_of(c)

            c = nt.OpCounter()
            p = nt.Polynomial(x.copy(), "truncated")
            nt.intt_gs_truncated(p, plan, c)
            vec[key + "_inttt"] = p.coeffs.copy()
            rec["inttt_counts"] = counts_of(c)

            # fused middle on the reference's own truncated spectra
            ah = nt.Polynomial(a.copy())
            bh = nt.Polynomial(b.copy())
            nt.ntt_ct_truncated(ah, plan)
            nt.ntt_ct_truncated(bh, plan)
            ch = np.empty(n, dtype=np.uint64)
            cnt = np.zeros(5, dtype=np.uint64)
            q, mode, mu, s_in, s_out = nt.nttcore._red_args(plan)
            backend.kernels().fused_middle(ah.coeffs, bh.coeffs, ch, plan.tw_fwd, q, mode,
                                           mu, s_in, s_out, cnt)
            vec[key + "_mid"] = ch
            rec["mid_counts"] = [int(v) for v in cnt]

        c = nt.OpCounter()
        vec[key + "_fused"] = nt.polymul_fused(nt.Polynomial(a.copy()),
                                               nt.Polynomial(b.copy()), plan, c)
        rec["fused_counts"] = counts_of(c)
        c = nt.OpCounter()
        vec[key + "_pntt"] = nt.polymul_ntt(nt.Polynomial(a.copy()),
                                            nt.Polynomial(b.copy()), plan, c)
        rec["pntt_counts"] = counts_of(c)
        vec[key + "_naive"] = nt.negacyclic_naive(a, b, plan.q)
        c = nt.OpCounter()
        nt.negacyclic_naive(a, b, plan.q, c)
        rec["naive_counts"] = counts_of(c)
        # alternative transform shapes (nttcore.py:189-497)
        if plan.log_n % 2 == 0:
            c = nt.OpCounter()
            p = nt.Polynomial(a.copy())
            nt.ntt_radix4(p, plan, c)
            vec[key + "_r4"] = p.coeffs.copy()
            rec["r4_counts"] = counts_of(c)
            c = nt.OpCounter()
            p = nt.Polynomial(x.copy(), "bit_reversed")
            nt.intt_radix4(p, plan, c)
            vec[key + "_ir4"] = p.coeffs.copy()
            rec["ir4_counts"] = counts_of(c)
        c = nt.OpCounter()
        p = nt.Polynomial(a.copy())
        nt.ntt_2d(p, plan, c)
        vec[key + "_2d"] = p.coeffs.copy()
        rec["2d_counts"] = counts_of(c)
        c = nt.OpCounter()
        p = nt.Polynomial(x.copy(), "vendor_2d")
        nt.ntt_2d_inv(p, plan, c)
        vec[key + "_2di"] = p.coeffs.copy()
        rec["2di_counts"] = counts_of(c)
        vec[key + "_2dperm"] = nt.ntt_2d_permutation(plan).astype(np.int64)
        vec[key + "_had"] = nt.hadamard(a, b, plan)
        f = int(rand(plan.q, 1, 4000 + n)[0])
        p = nt.Polynomial(a.copy())
        nt.scale_by(f, p, plan)
        vec[key + "_scale"] = p.coeffs.copy()
        rec["scale_factor"] = f
        cases.append(rec)
    out["vector_cases"] = cases
    np.savez_compressed(os.path.join(HERE, "vectors.npz"), **vec)

    # ---- large sizes: SHA-256 digests of reference outputs --------------
    big = []
    for n in (1 << 12, 1 << 13, 1 << 14, 1 << 15, 1 << 16, 1 << 17):
        plan = nt.build_plan(n, bits=60, seed=0)
        a = rand(plan.q, n, 11)
        b = rand(plan.q, n, 12)
        rec = {"n": n, "bits": 60, "seed": 0, "q": plan.q, "psi": plan.psi,
               "a_seed": 11, "b_seed": 12}
        p = nt.Polynomial(a.copy())
        nt.ntt_ct(p, plan)
        rec["ntt_sha"] = digest(p.coeffs)
        nt.intt_gs_scaled(p, plan)
        assert np.array_equal(p.coeffs, a)
        p = nt.Polynomial(a.copy())
        nt.ntt_ct_truncated(p, plan)
        rec["nttt_sha"] = digest(p.coeffs)
        x = rand(plan.q, n, 13)
        p = nt.Polynomial(x.copy(), "bit_reversed")
        nt.intt_gs(p, plan)
        rec["intt_x_seed"] = 13
        rec["intt_sha"] = digest(p.coeffs)
        c = nt.OpCounter()
        fused = nt.polymul_fused(nt.Polynomial(a), nt.Polynomial(b),
                                 nt.FusedPlan.from_plan(plan), c)
        rec["fused_sha"] = digest(fused)
        rec["fused_counts"] = counts_of(c)
        rec["fused_head"] = [int(v) for v in fused[:4]]
        big.append(rec)
        print("big", n, flush=True)
    out["large"] = big

    # ---- known answers --------------------------------------------------
    mod = nt.Modulus(994705409)
    out["named_triple"] = {"q": 994705409, "a": 994674970, "b": 994705408,
                           "want": nt.reduce_builtin(994674970 * 994705408, mod.q)}
    sinks = []
    for bits, passes in [(30, 1), (30, 2), (60, 3), (62, 1)]:
        q = nt.build_plan(2, bits=bits, seed=0).q
        a = rand(q, 4096, 50 + bits)
        b = rand(q, 4096, 60 + bits)
        m = nt.Modulus(q)
        for variant in ("builtin", "classical", "dhem", "proposed"):
            if variant == "dhem" and bits > 60:
                continue
            mode, mu, s_in, s_out = m.reduction_params(variant)
            s = backend.kernels().mulmod_loop(a, b, q, mode, mu, s_in, s_out, passes)
            sinks.append({"bits": bits, "q": q, "a_seed": 50 + bits, "b_seed": 60 + bits,
                          "n": 4096, "variant": variant, "passes": passes, "sink": int(s)})
    out["mulmod_loop"] = sinks

    # ---- Barrett-variant sweeps (_kernels.pyx:264-356) -------------------
    sweeps = []
    for q_lo, q_hi in [(3, 63), (3, 255), (200, 301)]:
        t = np.zeros((3, 4), dtype=np.uint64)
        mism, first = backend.kernels().sweep_exhaustive(q_lo, q_hi, t)
        sweeps.append({"kind": "exhaustive", "q_lo": q_lo, "q_hi": q_hi, "mism": int(mism),
                       "first": list(first) if first else None,
                       "tallies": [[int(v) for v in r] for r in t]})
    for bits, samples, seed in [(8, 100000, 0), (20, 100000, 1), (30, 100000, 2),
                                (60, 100000, 3), (61, 50000, 4), (62, 100000, 5),
                                (63, 50000, 6)]:
        t = np.zeros((3, 4), dtype=np.uint64)
        mism, first = backend.kernels().sweep_random(bits, samples, seed, t)
        sweeps.append({"kind": "random", "bits": bits, "samples": samples, "seed": seed,
                       "mism": int(mism), "first": list(first) if first else None,
                       "tallies": [[int(v) for v in r] for r in t]})
    out["sweeps"] = sweeps

    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
