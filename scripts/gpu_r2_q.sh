mkdir -p gpurun_out
for w in cfg5 cfg4b; do bash scripts/gpu_ab_multi.sh "base nst3 nst5c" 2 --workload $w; done
