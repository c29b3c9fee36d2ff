mkdir -p gpurun_out
for w in cfg3 cfg4a cfg4b cfg4 cfg5; do
  timeout 400 python bench.py --workload $w > gpurun_out/bench_${w}_final.json 2> gpurun_out/bench_${w}_final.err; echo "$w rc $? $(python scripts/show_bench.py gpurun_out/bench_${w}_final.json | cut -c1-150)"
done
