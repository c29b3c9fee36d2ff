mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_large_k_gpu.py tests/test_multirank_gpu.py -k "tiled or tc_ or split or left or ragged or cfg5 or companions or ranks" -q -x -p no:cacheprovider > gpurun_out/pytest_fin.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_fin.log)"
bash scripts/gpu_ab_multi.sh "cur orig" 2 --workload cfg5 | cut -c1-125
timeout 300 python scripts/tiled_phases.py 2147483648 65536 1 2>&1 | tail -8
