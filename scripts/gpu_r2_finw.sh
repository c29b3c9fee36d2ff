timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu_all.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu_all.log)"; grep -E "^FAILED" gpurun_out/pytest_gpu_all.log | head -5
for w in cfg4 cfg4d cfg4a cfg5; do for fw in 1 0; do
  TM_FIN_WHOLE=$fw timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "$w fw=$fw $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-120)"
done; done
