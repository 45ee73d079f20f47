# deferred layer join: tests, then bench A/B against the previous build (libtpipe_v0.so swapped in)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_realkernels.py tests/test_gpu_fullsize.py -x -q > gpurun_out/defer_tests.log 2>&1; echo "tests $?" >> gpurun_out/defer_tests.log
cp paper_2503_03182_b200/libtpipe.so /tmp/libtpipe_new.so
for r in 1 2; do
  cp paper_2503_03182_b200/libtpipe_v0.so paper_2503_03182_b200/libtpipe.so
  timeout 400 python bench.py --no-extras --steps 5 > gpurun_out/bench_defer_old.r$r.json 2>/dev/null
  cp /tmp/libtpipe_new.so paper_2503_03182_b200/libtpipe.so
  timeout 400 python bench.py --no-extras --steps 5 > gpurun_out/bench_defer_new.r$r.json 2>/dev/null
done
