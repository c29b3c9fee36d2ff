mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
for w in ${WLS:-cfg2 cfg4a cfg4}; do
timeout 300 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$w.log 2>&1; echo bench $w rc=$?
done
