mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/gc_kern.log 2>&1; echo "kern rc=$?" >> gpurun_out/gc_kern.log
timeout 600 python bench.py --steps 6 --warmup 3 --no-extras > gpurun_out/gc_bench.json 2> gpurun_out/gc_bench.err; echo "bench rc=$?" >> gpurun_out/gc_bench.err
timeout 600 python scripts/gemm_modes.py > gpurun_out/gc_modes.jsonl 2>&1
