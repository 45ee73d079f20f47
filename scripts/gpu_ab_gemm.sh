# A/B of the production GEMM against a reference build (paper_2503_03182_b200/libtpipe_v0.so)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k gemm > gpurun_out/ab_tests.log 2>&1; echo "tests $?" >> gpurun_out/ab_tests.log
for r in 1 2; do for L in libtpipe_v0.so libtpipe.so; do TPIPE_PROBE_LIB=$L timeout 200 python scripts/gemm_probe.py; done; done > gpurun_out/gemm_ab.jsonl 2> gpurun_out/gemm_ab.err
for s in fc1_fprop o_fprop fc2_dgrad; do TPIPE_GEMM_PROBE=0 timeout 100 python scripts/gemm_trace.py $s; done > gpurun_out/gemm_trace_ab.jsonl 2>> gpurun_out/gemm_ab.err
