mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -k "tiled_sparse or tc_one_cta_and_tiled or tc_engine_limbs" -q -x -p no:cacheprovider > gpurun_out/pytest_sparse.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_sparse.log)"
for i in 1 2; do for w in cfg4 cfg5; do for sp in 1 0; do
  TM_TILED_SPARSE=$sp timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "$i $w sparse=$sp $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-150)"
done; done; done
timeout 300 python scripts/tiled_phases.py 16777216 16384 64 2>&1 | tail -12
C="python bench.py --workload cfg4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
$C > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg4.csv $C > gpurun_out/ncu.log 2>&1; echo "ncu rc $?"
python scripts/show_launches.py gpurun_out/launches_cfg4.csv 2>&1 | tail -15
