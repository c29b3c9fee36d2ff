timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_large_k_gpu.py -k "tiled or tc_ or every_pair_int or split or left or ragged or cfg5 or companions or limbs" -q -x -p no:cacheprovider > gpurun_out/pytest_epi.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_epi.log)"
for w in cfg4 cfg5 cfg4c cfg4a; do bash scripts/gpu_ab_multi.sh "cur orig" 1 --workload $w | cut -c1-125; done
echo phases; timeout 300 python scripts/tiled_phases.py 16777216 16384 64 2>&1 | tail -9
