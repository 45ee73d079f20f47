# executed capacity (p = 8 virtual pipeline, 20 GiB per stage) with the final round-2 kernels
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TPIPE_CAPACITY_ONLY=1f1b,1f1b_r50,1f1b_full_recomp,tpipe,tpipe_trecomp,tpipe_all,tpipe_all_v3 timeout 3300 python bench.py --capacity-run > gpurun_out/r2_capacity_v6.json 2> gpurun_out/r2_capacity_v6.err
echo "rc $?" >> gpurun_out/r2_capacity_v6.err
