mkdir -p gpurun_out
bash scripts/gpu_ab_multi.sh "base orig a b c d" 1 --workload cfg4
