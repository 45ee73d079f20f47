set -x
mkdir -p gpurun_out
TPIPE_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 2 --warmup 3 --no-extras > gpurun_out/r2_bench_2rank_samegpu.json 2> gpurun_out/r2_bench_2rank_samegpu.err
for cfg in "c1 tpipe_trecomp 0 1 4 8" "c1 tpipe 5 1 2 4" "c1 tpipe 2 1 2 4" "cmid tpipe_trecomp 0 1 2 4" "cmid tpipe 5 1 1 2" "c1 tpipe_trecomp 0 0 2 4"; do
  for tool in memcheck synccheck racecheck; do
    tag=$(echo $cfg | tr ' ' '_')
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_step.py $cfg > gpurun_out/san_${tool}_${tag}.log 2>&1
    echo "$tool $tag rc=$?" >> gpurun_out/san_summary.txt
    tail -3 gpurun_out/san_${tool}_${tag}.log >> gpurun_out/san_summary.txt
  done
done
