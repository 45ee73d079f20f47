mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r2i_gputest.log
TPIPE_CAPACITY_ONLY=tpipe_all_v3 timeout 1200 python bench.py --capacity-run > gpurun_out/r2_capacity_v4.json 2> gpurun_out/r2_capacity_v4.err
timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 > gpurun_out/r2_workload_c3.json 2> gpurun_out/r2_workload_c3.err
timeout 1200 python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/r2_workload_c4.json 2> gpurun_out/r2_workload_c4.err
timeout 900 python bench.py --oracle-timing > gpurun_out/r2_oracle_timing.json 2> gpurun_out/r2_oracle_timing.err
