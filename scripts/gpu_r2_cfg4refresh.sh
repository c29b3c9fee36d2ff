mkdir -p gpurun_out
for w in cfg4 cfg4c cfg4d; do
  timeout 400 python bench.py --workload $w --no-cfg1 > gpurun_out/bench_${w}_final.json 2> gpurun_out/bench_${w}_final.err; echo "$w $(python scripts/show_bench.py gpurun_out/bench_${w}_final.json | cut -c1-160)"
done
