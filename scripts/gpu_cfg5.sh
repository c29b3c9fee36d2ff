mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -rf --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python bench.py --workload cfg5 --steps 20 --warmup 3 --e2e-steps 2 > gpurun_out/bench_cfg5.log 2>&1; echo bench cfg5 rc=$?
for w in cfg4 cfg2; do timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$w.log 2>&1; echo bench $w rc=$?; done
