cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/torchrun1.log 2>&1; echo "exit $?" >> gpurun_out/torchrun1.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/torchrun1_ref.log 2>&1; echo "exit $?" >> gpurun_out/torchrun1_ref.log
