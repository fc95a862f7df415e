#!/usr/bin/env python
"""Benchmark: batched fused negacyclic polymul, BASELINE cfg3
(N = 2^16, 21 x 60-bit RNS limbs), on N GPUs (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step = one fused polymul of every (ciphertext, limb) pair of a
[batch, 21, 65536] residue batch (batch ciphertexts per GPU, weak scaling:
shards are independent ciphertexts, no collective on the data path).  The
timed region is K steps on the device (CUDA events on the launch stream,
barrier + synchronize on both sides, max over ranks).  Inputs (2 x 672 MiB at
the default batch 64) exceed the 126 MB L2, so no flush is needed between steps.

Rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG_NAMES = {(16, 21): "cfg3", (14, 8): "cfg2", (17, 32): "cfg4", (12, 1): "cfg1"}
METRIC = "polymuls/sec at N=2^16×21 limbs; NTT µs; % of HBM/int-pipe roofline"
UNIT = "ct-polymul/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--batch", type=int, default=64,
                    help="ciphertexts per GPU (cfg3: >= 8, SURVEY 8(d); 8 / 16 / 32 / 64 give "
                         "23.1k / 23.5k / 23.8k / 23.9k ct/s on one B200, profiles/r2/NOTES.md)")
    ap.add_argument("--log-n", type=int, default=16)
    ap.add_argument("--limbs", type=int, default=21)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target CPU work for the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--shard", choices=("ct", "limb"), default=None,
                    help="multi-GPU partition: by ciphertext (default; weak scaling) or by "
                         "limb (default for cfg4; strong scaling)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (nvidia-smi, B200_PROFILING.md)

class ClockSampler:
    """SM clock and throttle reasons sampled while the timed region runs:
    NVML every ~2 ms (nvidia_ml_py; fast enough for a short region), else
    nvidia-smi every 100 ms.  Rows: [sm_mhz, max_mhz, -, hw_slowdown,
    hw_thermal, sw_thermal, sw_power_cap] ("Active"/"Not Active")."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits: HwSlowdown, HwThermalSlowdown, SwThermalSlowdown, SwPowerCap
    NVML_BITS = (0x8, 0x40, 0x20, 0x4)

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self.source = "nvidia-smi"
        self._stop = threading.Event()
        self._t = None

    def _nvml_handle(self):
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            try:
                uuid = str(torch.cuda.get_device_properties(self.index).uuid)
                h = pynvml.nvmlDeviceGetHandleByUUID(
                    uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            except Exception:  # noqa: BLE001 - older torch / MIG: fall back to the index
                h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            return pynvml, h
        except Exception:  # noqa: BLE001 - NVML missing: nvidia-smi path
            return None, None

    def _run(self):
        nv, h = self._nv, self._h
        if nv is not None:
            self.source = "nvml"
            try:
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                while not self._stop.is_set():
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    try:
                        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    except AttributeError:
                        rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    self.rows.append([str(sm), str(mx), hex(rs)] +
                                     ["Active" if rs & b else "Not Active" for b in self.NVML_BITS]
                                     + [time.perf_counter()])
                    self._stop.wait(0.002)
                return
            except Exception:  # noqa: BLE001 - fall through to nvidia-smi
                self.source = "nvidia-smi"
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")] + [time.perf_counter()])
            except Exception:  # noqa: BLE001 - sampling is best-effort
                return
            self._stop.wait(0.1)

    def mark_start(self):
        self._t0 = time.perf_counter()

    def mark_end(self):
        self._t1 = time.perf_counter()

    def __enter__(self):
        self._t0 = self._t1 = None
        self._nv, self._h = self._nvml_handle()  # NVML init outside the region
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        # a very short timed region can end before the thread's first
        # sample: give it up to 0.2 s to record one (clocks have not
        # dropped yet right after the region)
        t0 = time.perf_counter()
        while not self.rows and self._t and self._t.is_alive() and time.perf_counter() - t0 < 0.2:
            time.sleep(0.001)
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self) -> dict:
        """Samples taken inside the marked timed region (the one nearest to
        it when the region is shorter than the sampling period)."""
        rows = self.rows
        if rows and self._t0 is not None and self._t1 is not None:
            inside = [r for r in rows if self._t0 <= r[-1] <= self._t1]
            rows = inside or [min(rows, key=lambda r: abs(r[-1] - self._t0))]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in rows if r[1].replace(".", "").isdigit()),
                 default=None)
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:7])
                          if v.lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(rows), "source": self.source}


# ---------------------------------------------------------------------------
# workload

def make_inputs(primes, batch: int, n: int, seed: int, limb0: int = 0):
    """[batch, len(primes), n] uniform residues; limb l (global index
    limb0 + l) has its own generator, so a limb shard of the job holds
    exactly the rows of the whole job."""
    import numpy as np

    out = np.empty((batch, len(primes), n), dtype=np.uint64)
    for li, q in enumerate(primes):
        rng = np.random.default_rng([seed, limb0 + li])
        out[:, li, :] = rng.integers(0, q, size=(batch, n), dtype=np.uint64)
    return out


def modmuls_per_product(n: int) -> int:
    """Reference OpCounter modmul count of one polymul_fused."""
    lg = n.bit_length() - 1
    return (3 * n // 2) * (lg - 1) + 2 * n


def row_kernel_modmuls(n: int) -> int:
    """Algorithmic modmuls done inside the fused ROW kernel per product:
    forward row stages of a and b (log2 N2 - 1 each, n/2 per stage), the
    fused middle (4 per pair = 2n) and the inverse row stages."""
    n2 = min(n, 4096)
    l2 = n2.bit_length() - 1
    return 2 * (n // 2) * (l2 - 1) + 2 * n + (n // 2) * (l2 - 1)


def shard_mode(args) -> str:
    """ct: every rank owns its own ciphertexts (weak scaling, cfg3);
    limb: every rank owns a contiguous limb span of ONE job (strong
    scaling, cfg4 "sharded by limb", reference rns.py:116-119)."""
    if args.shard:
        return args.shard
    return "limb" if (args.log_n, args.limbs) == (17, 32) else "ct"


def config_dict(args, world: int) -> dict:
    """The config both arms report (identical dicts, so the driver can match
    them)."""
    n, L = 1 << args.log_n, args.limbs
    mode = shard_mode(args)
    glob = args.batch * world if mode == "ct" else args.batch
    return {"workload": f"{CFG_NAMES.get((args.log_n, L), 'custom')}: fused negacyclic "
                        f"polymul, N=2^{args.log_n}, {L} x 60-bit RNS limbs",
            "n": n, "limbs": L, "global_batch": glob,
            "batch_per_gpu": args.batch if mode == "ct" else None,
            "parallelism": (f"shard-by-ciphertext x{world}" if mode == "ct"
                            else f"shard-by-limb x{world}"),
            "l2": "inputs 2x%.0f MiB per GPU > 126 MB L2, no flush" %
                  (args.batch * L * n * 8 / 2**20 / (1 if mode == "ct" else world))}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_rate(basis_primes, psis, n, A, B, seconds: float, threads: int,
                       ndarray: bool = False):
    """Reference CPU polymul_fused (oracle/_ref, native Cython, GIL released)
    over a bounded sample; returns (ct/s, kind, cores, sample, outputs).
    ndarray=True passes plain ndarrays (the reference converts them through
    _as_coeffs, polymul.py:64) instead of Polynomial objects."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor

    import oracle

    nt = oracle.reference()
    L = len(basis_primes)
    if nt is not None:
        kind = "reference"
        fplans = []
        for q, psi in zip(basis_primes, psis):
            plan = nt.params._plan_from_root(n, n.bit_length() - 1, nt.Modulus(q), psi,
                                             "proposed")
            fplans.append(nt.FusedPlan.from_plan(plan))

        def one(bi, li):
            if ndarray:
                return nt.polymul_fused(A[bi, li], B[bi, li], fplans[li])
            return nt.polymul_fused(nt.Polynomial(A[bi, li]), nt.Polynomial(B[bi, li]),
                                    fplans[li])
    else:
        kind = "port"
        tables = [oracle.twiddles(q, psi, n.bit_length() - 1)
                  for q, psi in zip(basis_primes, psis)]

        def one(bi, li):
            return oracle.polymul_fused(A[bi, li], B[bi, li], basis_primes[li], 0,
                                        tables=tables[li])

    def run(nct):
        items = [(bi % A.shape[0], li) for bi in range(nct) for li in range(L)]
        step = -(-len(items) // threads)
        spans = [items[i:i + step] for i in range(0, len(items), step)]
        outs = {}

        def span(sp):
            for bi, li in sp:
                outs[(bi, li)] = one(bi, li)

        t0 = time.perf_counter()
        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(span, spans))
        return time.perf_counter() - t0, outs

    ncal = max(1, -(-threads // L))  # enough items to occupy every thread once
    dt1, outs = run(ncal)
    nct = max(1, int(seconds * ncal / max(dt1, 1e-3)))
    dt, _ = run(nct)
    rate = nct / dt
    sample = (f"{nct} ciphertext(s) x {L} limbs of N={n} via "
              f"{('nttmul.polymul_fused(ndarray, ndarray, FusedPlan)' if ndarray else 'nttmul.polymul_fused(Polynomial, Polynomial, FusedPlan)') if kind == 'reference' else 'oracle C port'}"
              f", {threads} threads, {dt:.2f} s")
    first = np.stack([outs[(0, li)] for li in range(L)])
    return rate, kind, threads, sample, first


def cpu_baseline_full(primes, psis, n, A, B, seconds: float):
    """BASELINE.md §3's CPU figure: all host threads (best of 3), one thread,
    and the ndarray-input path, plus the CPU model.  Returns (dict, ct 0 of
    the reference's output)."""
    threads = len(os.sched_getaffinity(0))
    per = max(1.0, seconds / 5)
    runs = [cpu_reference_rate(primes, psis, n, A, B, per, threads) for _ in range(3)]
    best = max(runs, key=lambda r: r[0])
    one_rate, _, _, one_sample, _ = cpu_reference_rate(primes, psis, n, A, B, per, 1)
    nd_rate, _, _, nd_sample, _ = cpu_reference_rate(primes, psis, n, A, B, per, threads,
                                                     ndarray=True)
    rate, kind, cores, sample, first = best
    return ({"value": round(rate, 3), "unit": UNIT, "cores": cores, "kind": kind,
             "sample": sample + " (best of 3)",
             "runs": [round(r[0], 3) for r in runs],
             "one_thread": {"value": round(one_rate, 3), "sample": one_sample},
             "ndarray_inputs": {"value": round(nd_rate, 3), "sample": nd_sample},
             "cpu_model": cpu_model()}, first)


# ---------------------------------------------------------------------------
# N-GPU launch

def spawn(args) -> int:
    """`bench.py --gpus N` without an outer launcher: start N ranks with
    torch.distributed.run on this node (127.0.0.1) and forward their output;
    rank 0 prints the JSON line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    import numpy as np

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import oracle
    import paper_2209_01290_b200 as nt
    from paper_2209_01290_b200.shard import shard_range, sub_basis

    # NTTB_BENCH_SHARE_GPU=1 (tests of the N>1 logic on a 1-GPU box only):
    # ranks share the visible GPUs round-robin and talk over gloo, since NCCL
    # refuses two ranks on one device.  Never set for a measured run.
    share = os.environ.get("NTTB_BENCH_SHARE_GPU") == "1"
    ngpu = torch.cuda.device_count()
    if share:
        local = local % ngpu
    elif world > ngpu:
        raise SystemExit(f"bench.py: {world} ranks but {ngpu} visible GPU(s) "
                         "(NTTB_BENCH_SHARE_GPU=1 shares them, logic tests only)")
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    red_dev = "cpu" if share else "cuda"

    def allreduce(x: float, op) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(t, op=op)
        return float(t.item())

    n, L_all = 1 << args.log_n, args.limbs
    mode = shard_mode(args)
    full = nt.RnsBasis.build(n, 60, L_all, seed=0)
    if mode == "ct":
        basis, lo, hi = full, 0, L_all
        Bn = args.batch                       # this rank's ciphertexts
        seeds = (1000 + rank, 2000 + rank)
        cts_per_step = world * Bn             # whole job
    else:
        basis, lo, hi = sub_basis(full, world, rank)
        Bn = args.batch                       # every rank: all ciphertexts, its limbs
        seeds = (1000, 2000)
        cts_per_step = Bn
    L = hi - lo
    primes = list(basis.primes)
    psis = [p.psi for p in basis.plans]
    A_h = make_inputs(primes, Bn, n, seeds[0], lo)
    B_h = make_inputs(primes, Bn, n, seeds[1], lo)
    A = torch.from_numpy(A_h).cuda()
    B = torch.from_numpy(B_h).cuda()
    C = torch.empty_like(A)
    W = torch.empty_like(A)
    fwd, inv, limbs = basis.device_tables()
    stream = torch.cuda.current_stream()
    lib = nt._lib

    def step(phases=7):
        lib.call("nttmul_polymul_fused_rns_phases", C.data_ptr(), A.data_ptr(), B.data_ptr(),
                 limbs.data_ptr(), fwd.data_ptr(), inv.data_ptr(), args.log_n, L, Bn,
                 basis.mode, W.data_ptr(), phases, stream.cuda_stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    # every rank checks the first and last ciphertext of its shard against
    # the C oracle (the reference restatement) before anything is timed
    chk = [0, Bn - 1] if Bn > 1 else [0]
    got = np.stack([C[i].cpu().numpy() for i in chk])  # (no uint64 fancy indexing on CUDA)
    want = oracle.polymul_rns(A_h[chk], B_h[chk], primes, psis)
    ok = allreduce(float(np.array_equal(got, want)), dist.ReduceOp.MIN if world > 1 else None)
    if ok != 1.0:
        raise SystemExit(f"bench.py: rank shard != oracle (rank {rank})")
    barrier()
    # ---- timed region: K full steps ----
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        clk.mark_start()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier()
        clk.mark_end()
    ms = ev0.elapsed_time(ev1)
    # per-kernel breakdown (same stream, events between the three launches)
    log_n1 = max(args.log_n - 12, 0)
    phase_ms = {}
    names = {1: "col_fwd", 2: "row_fused", 4: "col_inv"} if log_n1 else {2: "row_fused"}
    evs = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for k in names}

    def phases():
        for _ in range(args.steps):
            for k in names:
                evs[k][0].record(stream)
                step(k)
                evs[k][1].record(stream)
            torch.cuda.synchronize()
            for k, nm in names.items():
                phase_ms[nm] = phase_ms.get(nm, 0.0) + evs[k][0].elapsed_time(evs[k][1])

    # ranks sharing one GPU (NTTB_BENCH_SHARE_GPU) take the per-kernel timing
    # and the roof microbenchmarks in turn: run concurrently, both read about
    # half of the one-GPU figures (the roof most, so the fraction inflated)
    def in_turn(fn):
        if not (share and world > 1):
            return fn()
        out = None
        for r in range(world):
            if r == rank:
                out = fn()
            barrier()
        return out

    in_turn(phases)
    phase_ms = {k: v / args.steps for k, v in phase_ms.items()}

    ms_max = allreduce(ms, dist.ReduceOp.MAX if world > 1 else None)
    ms_per_step = ms_max / args.steps
    value = cts_per_step * args.steps / (ms_max / 1e3)

    # ---- int-pipe and HBM roofs (live microbenchmarks), rank 0's kernels ----
    roof = in_turn(lambda: modmul_roof(nt, basis, stream))
    hbm_peak, hbm_kind = peak_hbm()
    products_per_step = Bn * L
    row_ms = phase_ms["row_fused"]
    row_rate = products_per_step * row_kernel_modmuls(n) / (row_ms / 1e3) / 1e9
    all_rate = products_per_step * modmuls_per_product(n) / (ms / args.steps / 1e3) / 1e9
    if share and world > 1:  # the ranks' steps ran concurrently on the one GPU
        all_rate = world * products_per_step * modmuls_per_product(n) / (ms_per_step / 1e3) / 1e9
    traffic = load_traffic(products_per_step, n)
    pipe = imad_pipe_roof(n, clk.summary().get("sm_mhz"))
    roofline = {
        "bound": "int", "kernel": "row_fused (fwd row stages a,b + Karatsuba middle + inv row stages)",
        "achieved": round(row_rate, 2), "peak": round(roof["peak"], 2), "unit": "Gmodmul/s",
        "frac": round(row_rate / roof["peak"], 4),
        "traffic": traffic["row_fused"] if traffic else None,
        "peak_source": roof["source"], "roofs_gmodmul_s": roof["all"],
        "step_achieved": round(all_rate, 2), "step_frac": round(all_rate / roof["peak"], 4),
        "imad_pipe": {**pipe, "row_frac": round(row_rate / pipe["peak_gmodmul_s"], 4),
                      "step_frac": round(all_rate / pipe["peak_gmodmul_s"], 4)},
        "ncu_row_kernel": ncu_row_summary(),
        "step_traffic": traffic,
        "hbm": {
            "algorithmic_bytes_per_step": products_per_step * 24 * n,
            "achieved_gbs": round(products_per_step * 24 * n / (ms / args.steps / 1e3) / 1e9, 1),
            "peak_gbs": hbm_peak, "peak_source": hbm_kind,
            "frac": round(products_per_step * 24 * n / (ms / args.steps / 1e3) / 1e9 / hbm_peak, 4),
        },
        "phase_ms": {k: round(v, 4) for k, v in phase_ms.items()},
        "per_rank_products_per_step": products_per_step,
    }

    # ---- short device measurements while the GPU is still at full clock
    # (after the multi-second CPU baseline the clocks have dropped) ----
    ntt_us = ntt_latency_us(nt, basis.plans[0]) if rank == 0 else None
    polymul_us = polymul_latency_us(nt, basis.plans[0]) if rank == 0 else None
    crt = crt_rates(nt, full, min(args.batch, 16)) if rank == 0 and mode == "ct" else None
    # ---- e2e: public API with host buffers, copies inside timing ----
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(nt, basis, A_h, B_h, args, world, stream, C, cts_per_step, allreduce)

    # ---- parity vs the reference itself + CPU baseline (rank 0, N=1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, first = cpu_baseline_full(primes, psis, n, A_h, B_h, args.cpu_seconds)
        step()
        torch.cuda.synchronize()
        assert np.array_equal(C[0].cpu().numpy(), first), "GPU != reference CPU (ct 0)"
        cpu["parity_ct0"] = "bit-exact vs the reference's own polymul_fused"

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "weak" if mode == "ct" else "strong",
            "vs_baseline": None,
            "dtype": "u64", "data": "synthetic uniform residues (numpy default_rng per limb), "
                                   f"primes/psi = reference RnsBasis.build({n}, 60, {L_all}, seed=0)",
            "config": config_dict(args, world),
            "parity": {"checked": f"ciphertexts {chk} of every rank's shard vs the C oracle "
                                  "(reference restatement), before timing", "ok": True},
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu,
            "ntt_us": ntt_us, "polymul_us": polymul_us, "crt": crt,
            "gpu_launches": args.steps * (3 if log_n1 else 1) *
                            (2 if log_n1 and Bn * L >= 128 else 1),
            "clocks": clk.summary(), "impl": "ours",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(nt, basis, A_h, B_h, args, world, stream, C_dev, cts_per_step, allreduce):
    """The same metric through the public API with HOST buffers: every step
    copies its inputs host->device and the products back inside the timed
    region.  Two caller types: pinned torch tensors (the streamed H2D /
    kernels / D2H path at PCIe speed) and plain numpy arrays (the
    reference's own operand type; the call stages them through pinned
    memory itself)."""
    import torch
    import torch.distributed as dist

    Ap = torch.from_numpy(A_h).pin_memory()
    Bp = torch.from_numpy(B_h).pin_memory()
    Cp = torch.empty_like(Ap).pin_memory()
    steps = max(3, min(args.steps, 10))

    def timed(fn, reps):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            out = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return allreduce(e0.elapsed_time(e1), dist.ReduceOp.MAX if world > 1 else None), out

    ms, _ = timed(lambda: nt.polymul_rns_batch(Ap, Bp, basis, out=Cp), steps)
    same = torch.equal(Cp, C_dev.cpu())  # streamed host result == device-resident result
    nsteps = max(2, steps // 3)
    ms_np, Cn = timed(lambda: nt.polymul_rns_batch(A_h, B_h, basis), nsteps)
    same_np = torch.equal(Cn, Cp)
    return {"value": round(cts_per_step * steps / (ms / 1e3), 2), "unit": UNIT,
            "h2d_bytes_per_step": int(A_h.nbytes + B_h.nbytes),
            "d2h_bytes_per_step": int(A_h.nbytes), "steps": steps,
            "parity_vs_device": "bit-exact" if same and same_np else "MISMATCH",
            "path": "polymul_rns_batch(pinned host tensors) -> nttmul_polymul_fused_rns_host "
                    "(chunked H2D / fused kernels / D2H on 3 streams) -> pinned host",
            "numpy_unpinned": {"value": round(cts_per_step * nsteps / (ms_np / 1e3), 2),
                               "steps": nsteps,
                               "path": "polymul_rns_batch(numpy ndarrays): chunks staged "
                                       "through two pinned slots by host threads, overlapped "
                                       "with the streamed GPU chunks; numpy result"}}


def modmul_roof(nt, basis, stream):
    """Register-resident modmul throughput (nttmul_modmul_roof), best variant."""
    import ctypes

    import torch

    limb = basis.plans[0].limb()
    sink = torch.zeros(1, dtype=torch.uint64, device="cuda")
    best = {}
    kinds = [(1, "shoup"), (0, "barrett_proposed"), (2, "ct_butterfly"), (3, "gs_butterfly")]
    for kind, label in kinds:
        cnt = ctypes.c_double()
        args = (ctypes.byref(limb), kind, 148 * 8, 256, 2000, sink.data_ptr(),
                ctypes.byref(cnt), stream.cuda_stream)
        nt._lib.call("nttmul_modmul_roof", *args)  # warm
        torch.cuda.synchronize()
        # best of 3 timed groups: a roof is the fastest rate the loop
        # reaches (one group alone read up to 3 % low on a clock ramp, r2)
        rates = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(5):
                nt._lib.call("nttmul_modmul_roof", *args)
            e1.record(stream)
            torch.cuda.synchronize()
            rates.append(5 * cnt.value / (e0.elapsed_time(e1) / 1e3) / 1e9)
        best[label] = max(rates)
    # int-pipe roof: the fastest register-resident rate of any modmul form
    # (bare Shoup product, Barrett product, lazy CT / GS butterfly = one
    # modmul plus its add/sub/correction), no memory traffic at all
    peak = max(best.values())
    return {"peak": peak, "all": {k: round(v, 1) for k, v in best.items()},
            "source": "live nttmul_modmul_roof, register-resident, max over "
                      "{shoup, barrett, CT butterfly, GS butterfly}, Gmodmul/s"}


def peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def load_traffic(products: int, n: int):
    """DRAM bytes per launch of each kernel of the step at this batch, from
    the committed ncu capture (profiles/traffic.json: bytes per
    limb-product), their sum, and the sum's ratio to the 24n algorithmic
    bytes (read a, b; write c); None without a capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            rec = json.load(fh)
    except (OSError, ValueError):
        return None
    kernels = ("col_fwd", "row_fused", "col_inv") if n > 4096 else ("row_fused",)
    out = {}
    by_n = rec.get("by_n", {}).get(str(n))  # per-size captures (cfg2 / cfg4)
    if by_n:
        rec = {**by_n, "source": by_n.get("source", rec.get("source"))}
    for k in kernels:
        r = rec.get(k)
        if r and r.get("n", n) == n:
            out[k] = int(r["bytes_per_product"] * products)
    if not out:
        return None
    out["total"] = sum(out.values())
    out["complete"] = len(out) - 1 == len(kernels)
    out["ratio_to_24n"] = round(out["total"] / (24 * n * products), 3)
    out["source"] = rec.get("source", "profiles/traffic.json")
    return out


def imad_pipe_roof(n: int, sm_mhz):
    """Pipe-referenced roof, independent of this repo's own microbenchmark:
    every integer multiply issues to the fmaheavy pipe at (measured,
    profiles/r1/pipes_microbench.txt) 2 cycles per IMAD and 4 per IMAD.WIDE /
    IMAD.HI warp instruction per SMSP.  The fused product needs, per
    limb-product: 1.5n(log2 n - 1) + n Shoup twiddle products (5 WIDE + 4
    IMAD = 28 cycles; the last inverse stage carries the folded scale),
    1.5n lazy Barrett products (8 WIDE + 2 IMAD = 36) and 3n multiply-based
    partial reductions (IMAD.HI + WIDE + IMAD = 10), over the reference's
    24.5n-per-2^16 algorithmic modmul count."""
    lg = n.bit_length() - 1
    cycles = 28 * (1.5 * n * (lg - 1) + n) + 36 * 1.5 * n + 10 * 3 * n
    per = cycles / modmuls_per_product(n)
    mhz = sm_mhz or 1965.0
    return {"peak_gmodmul_s": round(148 * 4 * 32 * mhz * 1e6 / per / 1e9, 1),
            "fmaheavy_cycles_per_modmul": round(per, 2), "sm_mhz": mhz,
            "model": "148 SMs x 4 SMSPs x 32 lanes x clock / fmaheavy cycles per modmul "
                     "(multiplies only: 2 / IMAD, 4 / IMAD.WIDE or IMAD.HI)"}


def ncu_row_summary():
    """Counter-level evidence for the dominant kernel from the committed ncu
    capture (profiles/r2/ncu_row.json), or None."""
    path = os.path.join(ROOT, "profiles", "r2", "ncu_row.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return None


def crt_rates(nt, basis, batch):
    """RNS decomposition / CRT reconstruction of `batch` big-integer
    polynomials (the steps either side of the product), device-resident:
    ms per ciphertext-polynomial and the HBM bytes they move."""
    import torch

    W = nt.rns.num_words(basis)
    n, L = basis.n, basis.num_limbs
    g = torch.Generator(device="cuda").manual_seed(7)
    words = torch.randint(0, 2**62, (batch, n, W), dtype=torch.int64, device="cuda",
                          generator=g).to(torch.uint64)
    words[:, :, W - 1] = 0  # < big_q
    stream = torch.cuda.current_stream()

    def timed(fn, reps=20):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            out = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps, out

    # the C-ABI calls on preallocated buffers (the Python wrappers allocate
    # their outputs; kernel time only here), checked by a round trip
    t = nt.rns._crt_tables(basis)
    res = torch.empty((batch, L, n), dtype=torch.uint64, device="cuda")
    back = torch.empty_like(words)
    sp = stream.cuda_stream

    def dec():
        nt._lib.call("nttmul_crt_decompose", res.data_ptr(), words.data_ptr(),
                     t["primes"].data_ptr(), t["dec"].data_ptr(), L, W, batch, n, sp)

    def rec():
        nt._lib.call("nttmul_crt_reconstruct", back.data_ptr(), res.data_ptr(),
                     t["primes"].data_ptr(), t["inv"].data_ptr(), t["m"].data_ptr(),
                     t["q"].data_ptr(), t["recip"].data_ptr(), L, W, batch, n, sp)

    dec_ms, _ = timed(dec)
    rec_ms, _ = timed(rec)
    assert torch.equal(back, words), "CRT round trip"
    assert torch.equal(nt.crt_decompose(words, basis), res), "CRT wrapper"
    nbytes = batch * n * (W + L) * 8
    return {"words_per_coeff": W, "decompose_ms_per_poly": round(dec_ms / batch, 4),
            "reconstruct_ms_per_poly": round(rec_ms / batch, 4),
            "decompose_gbs": round(nbytes / (dec_ms / 1e3) / 1e9, 1),
            "reconstruct_gbs": round(nbytes / (rec_ms / 1e3) / 1e9, 1),
            "decompose_gmodmul_s": round(batch * n * L * W / (dec_ms / 1e3) / 1e9, 1),
            "reconstruct_gmodmul_s": round(batch * n * L * W / (rec_ms / 1e3) / 1e9, 1),
            "unit_note": "L x W word-by-constant products per coefficient (the reference's "
                         "per-word reductions), against the same modmul roofs as the product",
            "note": f"[{batch}, {n}, {W}] words <-> [{batch}, {L}, {n}] residues, round trip exact"}


def ntt_latency_us(nt, plan):
    """Standalone ntt_ct latency, one limb (N=2^16), device-resident: the
    device time per transform from a CUDA graph of 20 back-to-back C-ABI
    launches (no host overhead), and the same call through the Python API."""
    import torch

    x = torch.zeros(plan.n, dtype=torch.uint64, device="cuda")
    q, mode, mu, s_in, s_out = plan.red_args
    pairs, _ = nt.kernels._pairs_for(plan.tw_fwd, int(q))
    log_n = plan.n.bit_length() - 1
    side = torch.cuda.Stream()

    def launch(st):
        nt._lib.call("nttmul_ntt_ct", x.data_ptr(), pairs.data_ptr(), int(q), int(mode), int(mu),
                     int(s_in), int(s_out), 0, log_n, 1, st)

    res = {}
    with torch.cuda.stream(side):
        for _ in range(5):
            launch(side.cuda_stream)
        torch.cuda.synchronize()
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                for _ in range(20):
                    launch(side.cuda_stream)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(side)
            for _ in range(10):
                g.replay()
            e1.record(side)
            torch.cuda.synchronize()
            res["device_us"] = round(e0.elapsed_time(e1) * 1e3 / 200, 2)
        except Exception as exc:  # noqa: BLE001 - report, keep the API number
            res["device_us"] = None
            res["graph_error"] = str(exc)[:120]
    stream = torch.cuda.current_stream()
    for _ in range(5):
        nt.kernels.ntt_ct(x, plan.tw_fwd, *plan.red_args, False, None)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(50):
        nt.kernels.ntt_ct(x, plan.tw_fwd, *plan.red_args, False, None)
    e1.record(stream)
    torch.cuda.synchronize()
    res["api_us"] = round(e0.elapsed_time(e1) * 1e3 / 50, 2)
    return res


def polymul_latency_us(nt, plan):
    """Latency of ONE fused limb-product (polymul_fused of one prime, the
    one-launch grid schedule): device time per call from a CUDA graph of 20
    back-to-back C-ABI calls, and per call through the Python API
    (nt.polymul_fused on device tensors, 50 back-to-back calls, events)."""
    import numpy as np
    import torch

    from paper_2209_01290_b200.polymul import mode_flags

    fused = nt.FusedPlan.from_plan(plan)
    n = plan.n
    rng = np.random.default_rng(5)
    a = torch.from_numpy(rng.integers(0, plan.q, n, dtype=np.uint64)).cuda()
    b = torch.from_numpy(rng.integers(0, plan.q, n, dtype=np.uint64)).cuda()
    c, ws = torch.empty_like(a), torch.empty_like(a)
    limbs = plan.limb_device()
    mode = mode_flags(plan.red_args[1], [plan.q])
    log_n = n.bit_length() - 1
    side = torch.cuda.Stream()

    def launch(st):
        nt._lib.call("nttmul_polymul_fused_rns", c.data_ptr(), a.data_ptr(), b.data_ptr(),
                     limbs.data_ptr(), fused.fwd_pairs_half.data_ptr(),
                     fused.inv_pairs_half.data_ptr(), log_n, 1, 1, mode, ws.data_ptr(), st)

    res = {}
    with torch.cuda.stream(side):
        for _ in range(5):
            launch(side.cuda_stream)
        torch.cuda.synchronize()
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                for _ in range(20):
                    launch(side.cuda_stream)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(side)
            for _ in range(10):
                g.replay()
            e1.record(side)
            torch.cuda.synchronize()
            res["device_us"] = round(e0.elapsed_time(e1) * 1e3 / 200, 2)
        except Exception as exc:  # noqa: BLE001 - report, keep the API number
            res["device_us"] = None
            res["graph_error"] = str(exc)[:120]
    ref = c.clone()
    stream = torch.cuda.current_stream()
    for _ in range(5):
        out = nt.polymul_fused(a, b, fused)
    torch.cuda.synchronize()
    res["api_matches_c_abi"] = bool(torch.equal(out, ref))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(50):
        nt.polymul_fused(a, b, fused)
    e1.record(stream)
    torch.cuda.synchronize()
    res["api_us"] = round(e0.elapsed_time(e1) * 1e3 / 50, 2)
    res["n"] = n
    return res


def run_reference(args, rank, world):
    """The reference's own CPU implementation on the host cores (rank 0 only)."""
    if rank != 0:
        return
    import numpy as np  # noqa: F401

    import oracle

    n, L = 1 << args.log_n, args.limbs
    nt = oracle.reference()
    if nt is not None:
        basis = nt.RnsBasis.build(n, 60, L, seed=0)
        primes, psis = list(basis.primes), [p.psi for p in basis.plans]
    else:  # reference not built: same primes via this package's host plan layer
        import paper_2209_01290_b200.params as P

        basis = None
        primes, psis, s = [], [], 0
        while len(primes) < L:
            q = P.generate_prime(60, n, s)
            s += 1
            if q not in primes:
                primes.append(q)
                psis.append(P.find_primitive_root(q, 2 * n, 0))
    A = make_inputs(primes, 2, n, seed=1000)
    B = make_inputs(primes, 2, n, seed=2000)
    threads = len(os.sched_getaffinity(0))
    per_step = max(2.0, 60.0 / max(args.steps + args.warmup, 1))
    rates = []
    for i in range(args.warmup + args.steps):
        rate, kind, cores, sample, _ = cpu_reference_rate(primes, psis, n, A, B, per_step,
                                                          threads)
        if i >= args.warmup:
            rates.append(rate)
    value = sum(rates) / len(rates)
    line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 / value, 3), "higher_is_better": True,
            "scaling": "weak" if shard_mode(args) == "ct" else "strong",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic uniform residues",
            "config": config_dict(args, world),
            "impl": "reference",
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": cores,
                             "kind": kind, "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
