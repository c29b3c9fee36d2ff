# quick A/B of the default path vs the staged path + DRAM bytes of the hot kernel
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "cfg2 or cfg1 or tc_ or packed" > gpurun_out/pytest_ab.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_ab.log
for i in 1 2; do
timeout 120 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_fused.log 2>&1
TM_FUSED_TC=0 timeout 120 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_staged.log 2>&1
python scripts/show_bench.py gpurun_out/b_fused.log gpurun_out/b_staged.log
done
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fold_pm1 --csv $CMD 2>/dev/null | grep -E "dram|duration" | tail -3
