TM_LIB_VARIANT=s4 timeout 900 python -m pytest tests/test_parity_gpu.py -k "pm1 or packed or fold" -q -x -p no:cacheprovider > gpurun_out/pytest_s4.log 2>&1; echo "tests s4: $(tail -1 gpurun_out/pytest_s4.log)"
for i in 1 2; do for w in cfg5 cfg4b; do bash scripts/gpu_ab_multi.sh "cur s4 s16" 1 --workload $w | cut -c1-110; done; done
