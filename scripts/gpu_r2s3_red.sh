# session 3: tiled_reduce with 4 outputs per thread + packed-key max (A/B vs 1 output per thread), cfg4 epilogue vs nsp
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x -k "tiled or split or cfg5 or large or every_pair_int or all_limbs or multirank" > gpurun_out/s3r_pytest.log 2>&1; echo "tests: $(tail -1 gpurun_out/s3r_pytest.log)"
timeout 300 python scripts/tiled_phases.py 16777216 16384 64 > gpurun_out/s3_ph_cfg4b.txt 2>&1; echo "cfg4 ph rc $?"; cat gpurun_out/s3_ph_cfg4b.txt
for w in cfg5 cfg4c cfg4d; do
for i in 1 2 3; do
  for v in "" red1; do
    TM_LIB_VARIANT=$v timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
    echo "$w ${v:-new}: $(python scripts/show_bench.py gpurun_out/ab.log | cut -c1-150)"
  done
done
done
