# Full round check: smoke, GPU tests, default bench (with e2e + cpu_baseline), reference arm,
# ncu launch list, ncu --set full of the hot kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -q -rA --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fold_pm1_tma -s 3 -c 1 -o gpurun_out/ncu_full $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_full rc=$?
ncu -i gpurun_out/ncu_full.ncu-rep --page raw --csv > gpurun_out/ncu_full_raw.csv 2>/dev/null
