mkdir -p gpurun_out
timeout 1500 python bench.py --pipeline-replay > gpurun_out/r2_pipeline_replay_v1.json 2> gpurun_out/r2_pipeline_replay_v1.err
python scripts/gemm_shapes_once.py > gpurun_out/r2_gemm_shapes.jsonl 2>/dev/null
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 12 -c 12 -o gpurun_out/r2_gemm_full python scripts/gemm_shapes_once.py > /dev/null 2>&1
ncu -i gpurun_out/r2_gemm_full.ncu-rep --page raw --csv > gpurun_out/r2_gemm_full_raw.csv 2>/dev/null
python scripts/ncu_gemm_summary.py gpurun_out/r2_gemm_full_raw.csv gpurun_out/r2_gemm_shapes.jsonl > gpurun_out/r2_gemm_ncu_full_v1.jsonl
