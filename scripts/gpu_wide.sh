cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -k "wide_pair" -x -q > gpurun_out/wide_test.log 2>&1; echo "rc=$?" >> gpurun_out/wide_test.log
if grep -q "rc=0" gpurun_out/wide_test.log; then
  timeout 300 python scripts/gemm_wide_ab.py > gpurun_out/gemm_wide_ab.jsonl 2> gpurun_out/gemm_wide_ab.err
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 900 python bench.py --no-extras > gpurun_out/bench_noextras.json 2> gpurun_out/bench.err
fi
