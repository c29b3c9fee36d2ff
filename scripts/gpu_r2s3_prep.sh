# session 3: tiled_prep leftover fast path + per-kind plane loops (A/B vs HEAD build)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x -k "tiled or sparse or every_pair_int or cfg4 or cfg5 or randomized or large or all_limbs or split or multirank" > gpurun_out/s3p_pytest.log 2>&1; echo "tests: $(tail -1 gpurun_out/s3p_pytest.log)"
for w in cfg4 cfg5 cfg4c cfg4d; do
for i in 1 2; do
  for v in "" head; do
    TM_LIB_VARIANT=$v timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
    echo "$w ${v:-new}: $(python scripts/show_bench.py gpurun_out/ab.log | cut -c1-150)"
  done
done
done
C="python bench.py --workload cfg4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/s3p_launches_cfg4.csv $C > gpurun_out/s3p_ncu4.log 2>&1; echo "ncu launches rc $?"
