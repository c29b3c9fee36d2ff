mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_multirank_gpu.py tests/test_large_k_gpu.py -k "tiled or tc_ or split or cfg5 or companions or ranks" -q -x -p no:cacheprovider > gpurun_out/pytest_tile.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_tile.log)"
bash scripts/gpu_ab_multi.sh "cur orig" 2 --workload cfg5
for w in cfg4 cfg4c cfg4d; do bash scripts/gpu_ab_multi.sh "cur orig" 1 --workload $w; done
