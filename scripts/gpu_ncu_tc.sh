mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:corr_tc_kernel -s 2 -c 1 -o gpurun_out/ncu_tc $CMD > gpurun_out/ncu_tc.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_tc.log
