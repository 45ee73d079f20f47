# attention iteration: kernel parity tests, full-size sampled heads, timeline trace, warm timings
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "attention" > gpurun_out/attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/attn_tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "attention" >> gpurun_out/attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/attn_tests.log
timeout 300 python scripts/attn_trace.py > gpurun_out/attn_trace.txt 2>&1
timeout 300 python scripts/attn_time.py > gpurun_out/attn_time.jsonl 2>&1
