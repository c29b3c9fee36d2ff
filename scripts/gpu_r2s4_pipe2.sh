mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pipeline_gpu.py tests/test_multirank_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -5
B="python bench.py --no-cpu-baseline --no-cfg1 --e2e-steps 2"
for d in 1 2 3 2 3; do $B --pipeline $d > gpurun_out/p.json 2> gpurun_out/p.err || tail -5 gpurun_out/p.err; echo "cfg5 depth $d $(python scripts/show_bench.py gpurun_out/p.json | cut -c9-200)"; done
for w in cfg4 cfg4c cfg4b cfg4a cfg3 t2 cfg4d; do for d in 1 2 3; do $B --workload $w --pipeline $d > gpurun_out/p.json 2> gpurun_out/p.err || tail -5 gpurun_out/p.err; echo "$w depth $d $(python scripts/show_bench.py gpurun_out/p.json | cut -c9-200)"; done; done
