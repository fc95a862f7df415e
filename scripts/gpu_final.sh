# round-end style run: GPU tests, smoke, default bench, reference arm, launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_final.log 2>&1; echo "exit $?" >> gpurun_out/pytest_final.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_final.log 2>&1; echo "exit $?" >> gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "exit $?" >> gpurun_out/bench_final.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_final.log 2>&1; echo "exit $?" >> gpurun_out/bench_ref_final.log
