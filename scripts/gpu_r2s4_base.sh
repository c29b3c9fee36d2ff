# session-4 baseline: the GPU suite, smoke and the default line on the restored build
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu_s4.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu_s4.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s4.log 2>&1; echo "smoke rc $? $(tail -1 gpurun_out/smoke_s4.log)"
timeout 600 python bench.py > gpurun_out/bench_cfg5_s4.json 2> gpurun_out/bench_cfg5_s4.err; echo "cfg5 $(python scripts/show_bench.py gpurun_out/bench_cfg5_s4.json | cut -c1-170)"
for w in cfg2 cfg4 cfg3; do
  timeout 400 python bench.py --workload $w --no-cfg1 --no-cpu-baseline > gpurun_out/bench_${w}_s4.json 2> gpurun_out/bench_${w}_s4.err; echo "$w $(python scripts/show_bench.py gpurun_out/bench_${w}_s4.json | cut -c1-170)"
done
