mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "f32 or float or table2 or randomized or cfg3" > gpurun_out/f32_tests.log 2>&1; echo "tests: $(tail -1 gpurun_out/f32_tests.log)"
timeout 300 python bench.py --workload cfg3 --no-cpu-baseline > gpurun_out/cfg3.log 2>&1; python scripts/show_bench.py gpurun_out/cfg3.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_cfg3.log 2>&1; echo ncu rc $?
