# N>1 bench logic on one GPU (ranks share it over gloo; not a measurement) + torchrun N=1 both arms
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NTTB_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/torchrun2_share.log 2>&1; echo "exit $?" >> gpurun_out/torchrun2_share.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/torchrun2_ref.log 2>&1; echo "exit $?" >> gpurun_out/torchrun2_ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/torchrun1.log 2>&1; echo "exit $?" >> gpurun_out/torchrun1.log
