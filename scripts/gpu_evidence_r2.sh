# Round-2 evidence for the current kernels: ncu launch list of one C2 step,
# ncu --set full of the 12 layer GEMM shapes, compute-sanitizer on the new
# GEMM tile widths and the row-parallel LN backward.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
N=$(timeout 300 python scripts/profile_step.py 1 | awk '/launches/ {print $NF}' | tail -1)
echo "launches/step $N" > gpurun_out/launches_n.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s $N -c $N --csv --log-file gpurun_out/launches_v8.csv python scripts/profile_step.py 2 > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_v8.csv "ncu --metrics gpu__time_duration.sum --clock-control none -s $N -c $N python scripts/profile_step.py 2  (C2 1.3B T-Pipe p=1 m=32; window = all $N launches of step 1; cold-cache serialised: SHARES only)" > gpurun_out/launches_summary_v8.txt
timeout 300 python scripts/gemm_shapes_once.py > gpurun_out/gemm_shapes.jsonl 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:gemm_tc_kernel -s 12 -c 12 -o gpurun_out/gemm_full_v2 python scripts/gemm_shapes_once.py > gpurun_out/ncu_gemm_full.log 2>&1
ncu -i gpurun_out/gemm_full_v2.ncu-rep --page raw --csv > gpurun_out/gemm_full_v2_raw.csv 2>/dev/null
python scripts/ncu_gemm_summary.py gpurun_out/gemm_full_v2_raw.csv gpurun_out/gemm_shapes.jsonl > gpurun_out/r2_gemm_ncu_full_v2.jsonl 2>&1
for tool in memcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_kernels.py -x -q -k "wide_choice and 2048-2048-512 or rows_vs_staged and 37" > gpurun_out/san_r2b_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_r2b_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/san_r2b_${tool}.log >> gpurun_out/san_r2b_summary.txt
done
