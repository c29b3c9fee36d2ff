mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -k "tiled_sparse" -q -x -p no:cacheprovider > gpurun_out/pytest_epi.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_epi.log)"
bash scripts/gpu_ab_multi.sh "cur orig" 2 --workload cfg4 | cut -c1-125
TM_TILED_NT=64 bash scripts/gpu_ab_multi.sh "cur" 1 --workload cfg4 | cut -c1-125
for v in cur orig; do if [ $v = orig ]; then export TM_LIB_VARIANT=orig; fi; echo "phases $v"; timeout 300 python scripts/tiled_phases.py 16777216 16384 64 2>&1 | tail -9 | head -5; done
