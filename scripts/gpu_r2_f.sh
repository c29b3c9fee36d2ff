mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu.log)"
bash scripts/gpu_ab_multi.sh "base old_tiled" 2 --workload cfg5
for w in cfg4 cfg4b cfg4c cfg4d; do bash scripts/gpu_ab_multi.sh "base old_tiled" 1 --workload $w; done
TM_TC_TILED=1 timeout 200 python bench.py --workload cfg4b --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/t4b.log 2>&1; echo "cfg4b forced tiled: $(python scripts/show_bench.py gpurun_out/t4b.log | cut -c1-160)"
TM_TC_TILED=1 timeout 200 python bench.py --workload cfg4a --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/t4a.log 2>&1; echo "cfg4a forced tiled: $(python scripts/show_bench.py gpurun_out/t4a.log | cut -c1-160)"
timeout 200 python bench.py --workload cfg4a --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/b4a.log 2>&1; echo "cfg4a default: $(python scripts/show_bench.py gpurun_out/b4a.log | cut -c1-160)"
timeout 300 python scripts/tiled_phases.py 2147483648 65536 1 > gpurun_out/tiled_cfg5.txt 2>&1; cat gpurun_out/tiled_cfg5.txt
timeout 300 python scripts/tiled_phases.py 16777216 16384 64 > gpurun_out/tiled_cfg4.txt 2>&1; cat gpurun_out/tiled_cfg4.txt
