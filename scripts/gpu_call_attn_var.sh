mkdir -p gpurun_out
bash scripts/gpu_call_attn.sh
: > gpurun_out/attn_var.jsonl
for v in 0 4 8 10; do
  echo "{\"variant\": \"poly$v\"}" >> gpurun_out/attn_var.jsonl
  timeout 120 python scripts/attn_time.py --lib paper_2503_03182_b200/build/variants/libtpipe_p$v.so 1,2048,16,128 1,8192,16,128 >> gpurun_out/attn_var.jsonl 2>&1
done
