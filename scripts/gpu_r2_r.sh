mkdir -p gpurun_out
for w in cfg5 cfg4 cfg4a; do bash scripts/gpu_ab_multi.sh "base nst5c nst6c" 2 --workload $w; done
