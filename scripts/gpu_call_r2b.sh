# GPU tests (all) + capacity run after per-stage streams in the virtual pipeline
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/r2b_gputest.log
TPIPE_CAPACITY_ONLY=tpipe,tpipe_offload,tpipe_actoff,tpipe_actoff_offload,tpipe_all,1f1b_full_recomp,tpipe_trecomp timeout 1800 python bench.py --capacity-run > gpurun_out/r2_capacity_v2.json 2> gpurun_out/r2_capacity_v2.err
