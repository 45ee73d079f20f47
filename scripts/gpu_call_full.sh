# full validation: GPU test suite, smoke, default bench
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/full_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/full_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/full_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/full_smoke.log
timeout 900 python bench.py > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err; echo "rc=$?" >> gpurun_out/full_bench.err
