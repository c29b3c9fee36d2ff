mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider --durations=15 -rs > gpurun_out/pytest_gpu.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu.log)"; grep -E "SKIP|fused combine paths" gpurun_out/pytest_gpu.log | head
timeout 600 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "cfg5 $(python scripts/show_bench.py gpurun_out/bench_cfg5.json | cut -c1-200)"
for w in cfg2 cfg3 cfg4a cfg4b cfg4 cfg4c cfg4d t2; do timeout 400 python bench.py --workload $w --no-cpu-baseline --no-cfg1 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w $(python scripts/show_bench.py gpurun_out/bench_$w.json | cut -c1-200)"; done
