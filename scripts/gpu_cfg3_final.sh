mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_all.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu_all.log)"
timeout 400 python bench.py --workload cfg3 > gpurun_out/bench_cfg3_final.json 2> gpurun_out/bench_cfg3_final.err; echo "cfg3 $(python scripts/show_bench.py gpurun_out/bench_cfg3_final.json | cut -c1-150)"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg3_final.csv python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo "ncu cfg3 rc $?"
