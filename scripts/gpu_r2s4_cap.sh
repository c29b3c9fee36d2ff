# session-4 A/B: fold CTA cap under the two-stream pipeline
B="python bench.py --no-cpu-baseline --no-cfg1 --e2e-steps 0 --steps 100"
for c in 296 272 256 240 224; do TM_FOLD_SLOTS=$c $B > gpurun_out/p.json 2> gpurun_out/p.err || tail -3 gpurun_out/p.err; echo "cfg5 slots $c $(python scripts/show_bench.py gpurun_out/p.json | cut -c9-120)"; done
for c in 296 272 256 240 224 208; do TM_FOLD_DUAL=1 TM_FOLD_SLOTS=$c $B --workload cfg4 > gpurun_out/p.json 2> gpurun_out/p.err || tail -3 gpurun_out/p.err; echo "cfg4 dual slots $c $(python scripts/show_bench.py gpurun_out/p.json | cut -c9-160)"; done
for c in 296 256 224; do TM_FOLD_SLOTS=$c $B --workload cfg4b > gpurun_out/p.json 2> gpurun_out/p.err || tail -3 gpurun_out/p.err; echo "cfg4b slots $c $(python scripts/show_bench.py gpurun_out/p.json | cut -c9-160)"; done
for c in 296 256 224 192; do TM_FOLD_SLOTS=$c $B --workload cfg4c > gpurun_out/p.json 2> gpurun_out/p.err || tail -3 gpurun_out/p.err; echo "cfg4c slots $c $(python scripts/show_bench.py gpurun_out/p.json | cut -c9-160)"; done
