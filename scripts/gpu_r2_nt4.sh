timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -k "tiled or tc_ or every_pair_int" -q -x -p no:cacheprovider > gpurun_out/pytest_nt.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_nt.log)"
for w in cfg4 cfg4c cfg4d cfg5; do bash scripts/gpu_ab_multi.sh "cur orig" 1 --workload $w | cut -c1-125; done
