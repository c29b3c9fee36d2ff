# re-entry check: full GPU suite + smoke + default bench on the restored build
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu_all.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu_all.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $? $(tail -1 gpurun_out/smoke.log)"
timeout 600 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "cfg5 $(python scripts/show_bench.py gpurun_out/bench_cfg5.json | cut -c1-200)"
for w in cfg2 cfg3 cfg4 cfg4a; do
  timeout 400 python bench.py --workload $w --no-cfg1 > gpurun_out/bench_${w}.json 2> gpurun_out/bench_${w}.err; echo "$w $(python scripts/show_bench.py gpurun_out/bench_${w}.json | cut -c1-200)"
done
