mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -k "graph or side_stream" > gpurun_out/graph_tests.log 2>&1; echo "tests $?" >> gpurun_out/graph_tests.log
for r in 1 2; do for G in 0 1; do timeout 400 python bench.py --no-extras --graph $G --steps 5 > gpurun_out/bench_graph$G.r$r.json 2> gpurun_out/bench_graph$G.r$r.err; done; done
