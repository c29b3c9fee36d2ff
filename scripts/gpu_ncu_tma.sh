mkdir -p gpurun_out
./tools/stream_ceiling > gpurun_out/stream_ceiling.log 2>&1; echo ceiling rc=$?
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fold_pm1_tma|corr_fast" -s 2 -c 3 -o gpurun_out/prof_tma $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
