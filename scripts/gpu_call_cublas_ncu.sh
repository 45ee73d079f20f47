mkdir -p gpurun_out
timeout 900 ncu --set full --cache-control none --clock-control none -k regex:"nvjet|gemm_tc" -o gpurun_out/cmp_cublas python scripts/gemm_vs_cublas_ncu.py > gpurun_out/cmp_cublas.log 2>&1
echo rc=$? >> gpurun_out/cmp_cublas.log
ncu -i gpurun_out/cmp_cublas.ncu-rep --page raw --csv > gpurun_out/cmp_cublas_raw.csv 2>>gpurun_out/cmp_cublas.log
rm -f gpurun_out/cmp_cublas.ncu-rep
