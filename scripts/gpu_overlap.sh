mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
B="timeout 300 python bench.py --workload cfg2 --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0"
$B > gpurun_out/bench_cfg2.log 2>&1; echo bench rc=$?
TM_NO_OVERLAP=1 $B > gpurun_out/bench_cfg2_noov.log 2>&1; echo bench rc=$?
TM_OVERLAP_CHUNKS=2 $B > gpurun_out/bench_cfg2_c2.log 2>&1; echo bench rc=$?
TM_OVERLAP_CHUNKS=6 $B > gpurun_out/bench_cfg2_c6.log 2>&1; echo bench rc=$?
