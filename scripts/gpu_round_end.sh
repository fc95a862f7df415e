#!/usr/bin/env bash
# Round-end style evidence run on one B200 (what the driver runs, plus the
# extra configurations): GPU tests, smoke, default bench (cfg3), reference
# arm, cfg2 / cfg4 lines, the N=2 logic on the one GPU, cfg5 / schedule /
# latency sweeps.  Outputs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/re_pytest.log 2>&1; echo "exit $?" >> gpurun_out/re_pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/re_smoke.log 2>&1; echo "exit $?" >> gpurun_out/re_smoke.log
timeout 900 python bench.py > gpurun_out/re_bench.json 2> gpurun_out/re_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/re_bench_ref.json 2> gpurun_out/re_bench_ref.err
timeout 600 python bench.py --log-n 14 --limbs 8 --batch 64 --no-cpu-baseline > gpurun_out/re_bench_cfg2.json 2>&1
timeout 600 python bench.py --log-n 17 --limbs 32 --batch 8 --no-cpu-baseline > gpurun_out/re_bench_cfg4.json 2>&1
NTTB_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --no-cpu-baseline > gpurun_out/re_bench_share2.json 2>&1
timeout 600 python scripts/grid_sweep.py > gpurun_out/re_grid.jsonl 2>&1
timeout 300 python scripts/host_overhead.py > gpurun_out/re_host_overhead.jsonl 2>&1
timeout 600 python scripts/grid_fused_sweep.py > gpurun_out/re_grid_fused.jsonl 2>&1
timeout 600 python scripts/api_timing.py > gpurun_out/re_api_timing.jsonl 2>&1
timeout 900 python scripts/batched_xform.py > gpurun_out/re_batched.jsonl 2>&1
