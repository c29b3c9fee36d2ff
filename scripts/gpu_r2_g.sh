mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu.log)"
bash scripts/gpu_ab_multi.sh "base old_tiled" 1 --workload cfg5
for w in cfg4 cfg4b cfg4d; do bash scripts/gpu_ab_multi.sh "base old_tiled" 1 --workload $w; done
timeout 300 python scripts/tiled_phases.py 2147483648 65536 1 > gpurun_out/tiled_cfg5.txt 2>&1; cat gpurun_out/tiled_cfg5.txt
timeout 300 python scripts/tiled_phases.py 16777216 16384 64 > gpurun_out/tiled_cfg4.txt 2>&1; cat gpurun_out/tiled_cfg4.txt
C="python bench.py --workload cfg5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
$C > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"corr_tc_tiled|tiled_prep|tc_tiled_final" -s 3 -c 3 -o gpurun_out/prof_tiled5 $C > gpurun_out/ncu_t5.log 2>&1; echo "ncu rc $?"
