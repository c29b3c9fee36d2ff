# ncu of the correlation kernels at cfg5 (one pair, tiled) and cfg4 (K = 16384)
mkdir -p gpurun_out
for w in cfg5 cfg4; do
CMD="env TM_TC_TILED=1 TM_TILED_NT=32 python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"corr_tc" -s 1 -c 1 -o gpurun_out/ncu_corr_$w $CMD > gpurun_out/ncu_corr_$w.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/ncu_corr_$w.ncu-rep --page raw --csv > gpurun_out/ncu_corr_${w}_raw.csv 2>/dev/null
ncu -i gpurun_out/ncu_corr_$w.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_corr_${w}_sass.csv 2>/dev/null
done
