# round-end evidence with the final kernels: GPU tests, smoke, bench (graph steps),
# reference arm, ncu launch list of one step, ncu --set full of the 12 GEMM shapes
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/gputest.log
N=$(timeout 300 python scripts/profile_step.py 1 | awk '/launches/ {print $NF}' | tail -1)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s $N -c $N --csv --log-file gpurun_out/launches_v9.csv python scripts/profile_step.py 2 > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_v9.csv "ncu --metrics gpu__time_duration.sum --clock-control none -s $N -c $N python scripts/profile_step.py 2  (C2 1.3B T-Pipe p=1 m=32; window = all $N launches of step 1; cold-cache serialised: SHARES only)" > gpurun_out/launches_summary_v9.txt
timeout 300 python scripts/gemm_shapes_once.py > gpurun_out/gemm_shapes.jsonl 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:gemm_tc_kernel -s 12 -c 12 -o gpurun_out/gemm_full_v3 python scripts/gemm_shapes_once.py > gpurun_out/ncu_gemm_full.log 2>&1
ncu -i gpurun_out/gemm_full_v3.ncu-rep --page raw --csv > gpurun_out/gemm_full_v3_raw.csv 2>/dev/null
python scripts/ncu_gemm_summary.py gpurun_out/gemm_full_v3_raw.csv gpurun_out/gemm_shapes.jsonl > gpurun_out/r2_gemm_ncu_full_v3.jsonl 2>&1
