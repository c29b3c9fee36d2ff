# second refresh after the late NT / engine-threshold changes: full suite + the changed lines
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu_all.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu_all.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $? $(tail -1 gpurun_out/smoke.log)"
for w in cfg4 cfg4b cfg4c cfg4d; do
  timeout 400 python bench.py --workload $w --no-cfg1 > gpurun_out/bench_${w}_final.json 2> gpurun_out/bench_${w}_final.err; echo "$w $(python scripts/show_bench.py gpurun_out/bench_${w}_final.json | cut -c1-170)"
done
timeout 600 python bench.py > gpurun_out/bench_cfg5_final.json 2> gpurun_out/bench_cfg5_final.err; echo "cfg5 $(python scripts/show_bench.py gpurun_out/bench_cfg5_final.json | cut -c1-170)"
