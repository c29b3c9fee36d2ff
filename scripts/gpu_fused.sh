mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python bench.py --workload cfg2 --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_cfg2.log 2>&1; echo bench rc=$?
TM_NO_FUSED=1 timeout 300 python bench.py --workload cfg2 --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_cfg2_nofused.log 2>&1; echo bench rc=$?
