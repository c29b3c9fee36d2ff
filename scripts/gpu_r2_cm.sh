timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_large_k_gpu.py -k "tiled or tc_ or every_pair_int or block or limbs or cfg4 or companions" -q -x -p no:cacheprovider > gpurun_out/pytest_cm.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_cm.log)"; grep -E "^FAILED" gpurun_out/pytest_cm.log | head -3
for i in 1 2; do for w in cfg4 cfg4c cfg4d; do for cm in 1 0; do
  TM_COUNTS_MODE=$cm timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "$i $w cm=$cm $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-120)"
done; done; done
