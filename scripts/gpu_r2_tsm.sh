timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -k "tiled or every_pair_int" -q -x -p no:cacheprovider > gpurun_out/pytest_tsm.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_tsm.log)"
bash scripts/gpu_ab_multi.sh "cur orig" 2 --workload cfg4 | cut -c1-125
TM_TILED_NT=64 TM_TILED_NCR=1 bash scripts/gpu_ab_multi.sh "cur" 1 --workload cfg4 | cut -c1-125
for nt in 32 64; do echo "phases nt=$nt"; TM_TILED_NT=$nt TM_TILED_NCR=1 timeout 300 python scripts/tiled_phases.py 16777216 16384 64 2>&1 | tail -7; done
