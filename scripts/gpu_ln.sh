cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "layernorm or colsum" -x -q > gpurun_out/ln_test.log 2>&1; echo "rc=$?" >> gpurun_out/ln_test.log
if grep -q "rc=0" gpurun_out/ln_test.log; then
  timeout 300 python -c "import bench, json; print(json.dumps(bench.hbm_kernels(bench.C2, 6538.3)))" > gpurun_out/hbm_kernels.json 2>&1
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 900 python bench.py --no-extras > gpurun_out/bench_noextras.json 2> gpurun_out/bench.err
fi
