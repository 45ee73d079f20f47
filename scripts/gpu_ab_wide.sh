# 240/224-wide tiles on vs off, same library, same box
mkdir -p gpurun_out
for r in 1 2; do for W in 0 1; do GEMM_WIDE=$W TPIPE_PROBE_LIB=libtpipe.so timeout 200 python scripts/gemm_probe.py; done; done > gpurun_out/gemm_ab.jsonl 2> gpurun_out/gemm_ab.err
for s in fc1_fprop fc1_wgrad; do TPIPE_GEMM_PROBE=0 timeout 100 python scripts/gemm_trace.py $s; done > gpurun_out/gemm_trace_ab.jsonl 2>> gpurun_out/gemm_ab.err
