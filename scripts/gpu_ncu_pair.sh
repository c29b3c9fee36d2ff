mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"corr_pair|fold_pm1_tma" -s 2 -c 2 -o gpurun_out/prof_pair $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
