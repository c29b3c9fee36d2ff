# full GPU suite + the cfg4 / cfg5 lines on the current build
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu_all.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu_all.log)"
for w in ${WL:-cfg5 cfg4}; do
  timeout 400 python bench.py --workload $w --no-cfg1 > gpurun_out/bench_${w}.json 2> gpurun_out/bench_${w}.err; echo "$w $(python scripts/show_bench.py gpurun_out/bench_${w}.json | cut -c1-200)"
done
