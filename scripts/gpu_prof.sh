# parity + bench + ncu launch list + one full ncu capture of the hot kernels
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python bench.py --steps 100 --warmup 10 --cpu-seconds 5 > gpurun_out/bench.log 2>&1; echo bench rc=$?
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo ncu1 rc=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fold_pm1|corr_fast|fold_finalize" -s 3 -c 3 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
