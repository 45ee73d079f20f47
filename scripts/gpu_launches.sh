cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
N=$(timeout 300 python scripts/profile_step.py 1 | awk '/launches/ {print $NF}' | tail -1)
echo "launches/step $N" > gpurun_out/launches_n.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s $N -c $N --csv --log-file gpurun_out/launches_v5.csv python scripts/profile_step.py 2 > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_v5.csv "ncu --metrics gpu__time_duration.sum --clock-control none -s $N -c $N python scripts/profile_step.py 2  (C2 1.3B T-Pipe p=1 m=32; window = all $N launches of step 1; cold-cache serialised: SHARES only)" > gpurun_out/launches_summary_v5.txt
