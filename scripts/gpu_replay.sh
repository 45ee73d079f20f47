cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --pipeline-replay > gpurun_out/replay.json 2> gpurun_out/replay.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
