mkdir -p gpurun_out
TPIPE_CAPACITY_ONLY=1f1b,1f1b_r50,1f1b_full_recomp,tpipe,tpipe_trecomp,tpipe_all,tpipe_all_v3 timeout 3000 python bench.py --capacity-run --cap-p 2 --cap-budget-gib 80 > gpurun_out/r2_capacity_p2_80g.json 2> gpurun_out/r2_capacity_p2_80g.err
