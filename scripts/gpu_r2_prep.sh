mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_large_k_gpu.py tests/test_fullsize_gpu.py -k "tiled or tc_ or split or left or ragged or every_pair_int or cfg5 or limbs" -q -x -p no:cacheprovider > gpurun_out/pytest_prep.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_prep.log)"
for w in cfg5 cfg4 cfg4c; do bash scripts/gpu_ab_multi.sh "cur orig" 1 --workload $w | cut -c1-125; done
