timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_large_k_gpu.py -k "tiled or tc_ or every_pair_int or split or limbs or companions" -q -x -p no:cacheprovider > gpurun_out/pytest_nb.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_nb.log)"; grep -E "^FAILED" gpurun_out/pytest_nb.log | head -3
for i in 1 2; do for w in cfg4 cfg4b; do for nb in 3 2; do
  TM_TILED_NB=$nb timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "$i $w nb=$nb $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-130)"
done; done; done
echo phases-cfg4; timeout 300 python scripts/tiled_phases.py 16777216 16384 64 2>&1 | tail -10 | head -5
