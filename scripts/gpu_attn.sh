cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 120 python scripts/attn_probe.py 1 300 2 128 > gpurun_out/attn_probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/attn_probe.log
if grep -q "probe rc=0" gpurun_out/attn_probe.log; then
  timeout 400 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -k "attention" -x -q > gpurun_out/attn_test.log 2>&1; echo "rc=$?" >> gpurun_out/attn_test.log
  timeout 300 python scripts/attn_time.py 1,2048,16,128 1,8192,32,128 2,2048,32,64 > gpurun_out/attn_time.jsonl 2>&1
  if grep -q "rc=0" gpurun_out/attn_test.log; then
    timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
    timeout 900 python bench.py --no-extras > gpurun_out/bench_noextras.json 2> gpurun_out/bench.err
  fi
fi
