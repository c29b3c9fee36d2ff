mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-cfg1 --e2e-steps 2"
for r in 1 2; do $B > gpurun_out/p.json 2> gpurun_out/p.err || tail -5 gpurun_out/p.err; echo "cfg5 $(python scripts/show_bench.py gpurun_out/p.json | cut -c9-200)"; done
cp gpurun_out/p.json gpurun_out/bench_cfg5_pipe.json
for w in cfg4 cfg3 cfg2; do $B --workload $w > gpurun_out/p.json 2> gpurun_out/p.err || tail -5 gpurun_out/p.err; echo "$w $(python scripts/show_bench.py gpurun_out/p.json | cut -c9-200)"; done
