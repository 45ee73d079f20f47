mkdir -p gpurun_out
: > gpurun_out/san2_summary.txt
for cfg in "cmid12 tpipe_trecomp 5 1 2 4 3 0" "cmid12 1f1b_full_recomp 0 1 2 4 2 3" "cmid tpipe 0 1 1 2 2 0" "cmid12 interleave_trecomp 0 1 2 4 3 0"; do
  for tool in memcheck racecheck synccheck; do
    tag=$(echo $cfg | tr ' ' '_')
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_step.py $cfg > gpurun_out/san2_${tool}_${tag}.log 2>&1
    echo "$tool $tag rc=$?" >> gpurun_out/san2_summary.txt
    tail -2 gpurun_out/san2_${tool}_${tag}.log >> gpurun_out/san2_summary.txt
  done
done
