mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r2k_gputest.log
timeout 1200 python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/r2_workload_c4.json 2> gpurun_out/r2_workload_c4.err
timeout 600 python bench.py --no-extras --steps 10 > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1
