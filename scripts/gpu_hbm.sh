cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file gpurun_out/hbm_ncu.csv -k regex:'ln_|reduce_parts|colsum|ce_|adamw' python scripts/hbm_kernels_once.py > gpurun_out/hbm_once.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
