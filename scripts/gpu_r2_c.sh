mkdir -p gpurun_out
bash scripts/gpu_ab_multi.sh "base nst5 nst6 r560" 3 --workload cfg5
for nt in 32 64; do TM_TILED_NT=$nt timeout 200 python bench.py --workload cfg5 --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/nt$nt.log 2>&1; echo "NT=$nt $(python scripts/show_bench.py gpurun_out/nt$nt.log | cut -c1-160)"; done
bash scripts/gpu_ab_multi.sh "base nst5" 2 --workload cfg4
