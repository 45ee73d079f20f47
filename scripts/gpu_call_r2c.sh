mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/r2c_gputest.log
timeout 600 python bench.py --no-extras --steps 10 > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
