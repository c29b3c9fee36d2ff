# session 3 baseline: fresh-container build, whole GPU suite, default bench, cfg3 line + cfg3 launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -x > gpurun_out/s3_pytest_gpu.log 2>&1; echo "tests: $(tail -1 gpurun_out/s3_pytest_gpu.log)"
timeout 600 python bench.py > gpurun_out/s3_bench_cfg5.json 2> gpurun_out/s3_bench_cfg5.err; echo "cfg5 $(python scripts/show_bench.py gpurun_out/s3_bench_cfg5.json | cut -c1-200)"
timeout 400 python bench.py --workload cfg3 --no-cfg1 --no-cpu-baseline > gpurun_out/s3_bench_cfg3.json 2> gpurun_out/s3_bench_cfg3.err; echo "cfg3 $(python scripts/show_bench.py gpurun_out/s3_bench_cfg3.json | cut -c1-200)"
C="python bench.py --workload cfg3 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/s3_launches_cfg3.csv $C > gpurun_out/s3_ncu.log 2>&1; echo "ncu rc $?"
