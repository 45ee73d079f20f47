mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_realkernels.py -q -x -k multichunk 2>&1 | tail -30 > gpurun_out/r2h_mc.log
TPIPE_CAPACITY_ONLY=tpipe_all_v3,tpipe_all timeout 1500 python bench.py --capacity-run > gpurun_out/r2_capacity_v3.json 2> gpurun_out/r2_capacity_v3.err
