timeout 1500 python -m pytest tests/test_fullsize_gpu.py tests/test_parity_gpu.py -k "every_pair_int or tiled or tc_ or cfg2" -q -x -p no:cacheprovider > gpurun_out/pytest_4b.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_4b.log)"
for i in 1 2; do for w in cfg4b; do
  timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "$i $w $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-130)"
done; done
