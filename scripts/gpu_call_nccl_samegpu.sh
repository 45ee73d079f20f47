# Does NCCL accept two ranks on one GPU? (evidence for DESIGN §8)
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/nccl_samegpu.log 2>&1
NCCL_DEBUG=WARN TPIPE_BENCH_SAME_GPU=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --no-extras --transport nccl \
  >> gpurun_out/nccl_samegpu.log 2>&1
echo "rc=$?" >> gpurun_out/nccl_samegpu.log
