for g in 296 264 240 216 192 148; do
  TM_FOLD_GRID=$g timeout 200 python bench.py --workload cfg5 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "grid=$g $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-120)"
done
for g in 296 240 192; do
  TM_FOLD_GRID=$g timeout 200 python bench.py --workload cfg4 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "cfg4 grid=$g $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-120)"
done
