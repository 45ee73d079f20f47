mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_realkernels.py -q -k "partial_recompute or planned" 2>&1 | tail -8 > gpurun_out/r2l_gputest.log
TPIPE_CAPACITY_ONLY=1f1b_r50,1f1b_full_recomp,tpipe_all,tpipe_all_v3,tpipe,tpipe_trecomp timeout 2400 python bench.py --capacity-run > gpurun_out/r2_capacity_v5.json 2> gpurun_out/r2_capacity_v5.err
