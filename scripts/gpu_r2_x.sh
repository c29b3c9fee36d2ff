mkdir -p gpurun_out
bash scripts/gpu_ab_multi.sh "base pre" 3 --workload cfg2
bash scripts/gpu_ab_multi.sh "base pre" 1 --workload cfg5
