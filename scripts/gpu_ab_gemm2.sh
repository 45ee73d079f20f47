# A/B of the production GEMM library against a variant build (libtpipe_v0.so), GEMM tests first
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k gemm > gpurun_out/ab_tests.log 2>&1; echo "tests $?" >> gpurun_out/ab_tests.log
export GEMM_PROBE_SHAPES=${GEMM_PROBE_SHAPES:-fc2_wgrad,fc1_wgrad,o_wgrad,qkv_wgrad,head_wgrad,fc1_fprop}
for r in 1 2 3; do for L in libtpipe_v0.so libtpipe.so; do TPIPE_PROBE_LIB=$L timeout 200 python scripts/gemm_probe.py; done; done > gpurun_out/gemm_ab.jsonl 2> gpurun_out/gemm_ab.err
