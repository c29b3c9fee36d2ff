mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fold_pm1_tma -s 3 -c 1 -o gpurun_out/ncu_fused $CMD > gpurun_out/ncu_fused.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/ncu_fused.ncu-rep --page raw --csv > gpurun_out/ncu_fused_raw.csv 2>/dev/null
ncu -i gpurun_out/ncu_fused.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_fused_sass.csv 2>/dev/null
