mkdir -p gpurun_out
export GEMM_WIDE=0
for r in 1 2; do for P in 0 16; do TPIPE_GEMM_PROBE=$P timeout 200 python scripts/gemm_probe.py; done; done > gpurun_out/gemm_ab.jsonl 2> gpurun_out/gemm_ab.err
for s in fc1_fprop fc2_wgrad; do TPIPE_GEMM_PROBE=16 timeout 100 python scripts/gemm_trace.py $s; done > gpurun_out/gemm_trace_ab.jsonl 2>> gpurun_out/gemm_ab.err
