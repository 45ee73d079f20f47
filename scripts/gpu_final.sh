cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py -k "partition_offload" -x -q > gpurun_out/compose_test.log 2>&1; echo "rc=$?" >> gpurun_out/compose_test.log
N=$(timeout 300 python scripts/profile_step.py 1 | awk '/launches/ {print $NF}' | tail -1)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s $N -c $N --csv --log-file gpurun_out/launches_v6.csv python scripts/profile_step.py 2 > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_v6.csv "ncu --metrics gpu__time_duration.sum --clock-control none -s $N -c $N python scripts/profile_step.py 2  (C2 1.3B T-Pipe p=1 m=32; window = all $N launches of step 1; cold-cache serialised: SHARES only)" > gpurun_out/launches_summary_v6.txt
