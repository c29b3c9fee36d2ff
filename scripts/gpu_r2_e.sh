mkdir -p gpurun_out
bash scripts/gpu_ab_multi.sh "base noef nocomp nocomp_nst5" 2 --workload cfg5
bash scripts/gpu_ab_multi.sh "base noef nocomp" 1 --workload cfg4
bash scripts/gpu_ab_multi.sh "base noef" 1 --workload cfg2
