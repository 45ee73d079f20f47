mkdir -p gpurun_out
# 1) the N-rank bench path with DP x PP on one GPU (4 processes: pp 2 x dp 2)
TPIPE_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --pp 2 --steps 2 --warmup 3 --no-extras > gpurun_out/r2_bench_dp2pp2_samegpu.json 2> gpurun_out/r2_bench_dp2pp2_samegpu.err
# 2) launch list of one step of the bench workload (last step of 2)
L=$(python scripts/profile_step.py 1 2>/dev/null | grep launches | awk '{print $NF}')
echo "launches/step $L" > gpurun_out/r2_launch_count.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c $((2 * L + 64)) --csv --log-file gpurun_out/r2_launches_v7.csv python scripts/profile_step.py 2 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/r2_launches_v7.csv "ncu --metrics gpu__time_duration.sum --clock-control none python scripts/profile_step.py 2 (C2 1.3B T-Pipe p=1 m=32, fused K8 head); last $L launches = step 1; cold-cache serialised: SHARES only" $L > gpurun_out/r2_launches_summary_v7.txt
# 3) the default bench line
timeout 1200 python bench.py > gpurun_out/r2_bench_full_v1.json 2> gpurun_out/r2_bench_full_v1.err
