mkdir -p gpurun_out
CMD="python bench.py --workload cfg5 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"corr_tc_tiled|tc_tiled_finish" -s 2 -c 2 -o gpurun_out/ncu_tiled $CMD > gpurun_out/ncu_tiled.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/ncu_tiled.ncu-rep --page raw --csv > gpurun_out/ncu_tiled_raw.csv 2>/dev/null
ncu -i gpurun_out/ncu_tiled.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_tiled_sass.csv 2>/dev/null
