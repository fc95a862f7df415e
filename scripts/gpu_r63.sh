# round-1 evidence refresh: tests, smoke, bench (both arms), launch list, ncu full
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r63.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r63.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_r63.log 2>&1; echo "exit $?" >> gpurun_out/smoke_r63.log
timeout 900 python bench.py > gpurun_out/bench_r63.log 2>&1; echo "exit $?" >> gpurun_out/bench_r63.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r63.log 2>&1; echo "exit $?" >> gpurun_out/bench_ref_r63.log
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r63.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_r63.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"row_kernel|col_kernel" -c 3 -o /tmp/prof_r63 \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --batch 8 > gpurun_out/ncu_r63.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_r63.log
ncu -i /tmp/prof_r63.ncu-rep --page raw --csv > gpurun_out/ncu_r63_raw.csv 2>&1
ncu -i /tmp/prof_r63.ncu-rep --page details --csv > gpurun_out/ncu_r63_details.csv 2>&1
ncu -i /tmp/prof_r63.ncu-rep --page source --csv -k regex:row_kernel > gpurun_out/ncu_r63_row_source.csv 2>&1
ls -la /tmp/prof_r63.ncu-rep >> gpurun_out/ncu_r63.log
sz=$(stat -c %s /tmp/prof_r63.ncu-rep); [ "$sz" -lt 40000000 ] && cp /tmp/prof_r63.ncu-rep gpurun_out/
du -sh gpurun_out >> gpurun_out/ncu_r63.log
timeout 900 python scripts/ntt_sweep.py --out gpurun_out/cfg5_sweep_r63.jsonl > gpurun_out/cfg5_r63.log 2>&1
timeout 600 python bench.py --log-n 17 --limbs 32 --batch 8 --cpu-seconds 5 > gpurun_out/bench_cfg4_r63.log 2>&1
timeout 600 python bench.py --log-n 14 --limbs 8 --batch 64 --cpu-seconds 5 > gpurun_out/bench_cfg2_r63.log 2>&1
