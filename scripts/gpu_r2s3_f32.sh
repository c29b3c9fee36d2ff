# session 3: fp32 fold group-combined partials + template-first ordering; parity then same-box A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x -k "f32 or cfg3 or block or multi_moduli or table2 or randomized" > gpurun_out/s3f_pytest.log 2>&1; echo "tests: $(tail -1 gpurun_out/s3f_pytest.log)"
for w in cfg3 t2; do
for i in 1 2; do
  for v in "" f32old tlate f32one; do
    TM_LIB_VARIANT=$v timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
    echo "$w ${v:-new}: $(python scripts/show_bench.py gpurun_out/ab.log | cut -c1-150)"
  done
done
done
C="python bench.py --workload cfg3 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/s3f_launches_cfg3.csv $C > gpurun_out/s3f_ncu.log 2>&1; echo "ncu rc $?"
