mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_all.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu_all.log)"
for w in cfg5 cfg4 cfg4b; do
  timeout 400 python bench.py --workload $w > gpurun_out/bench_${w}_final.json 2> gpurun_out/bench_${w}_final.err; echo "$w $(python scripts/show_bench.py gpurun_out/bench_${w}_final.json | cut -c1-150)"
done
