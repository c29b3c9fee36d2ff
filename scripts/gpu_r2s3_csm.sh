# session 3: sparse corrections computed by the epilogue warps during the MMA loop (A/B vs TM_NO_CSM)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x -k "tiled or sparse or every_pair_int or cfg4 or randomized" > gpurun_out/s3c_pytest.log 2>&1; echo "tests: $(tail -1 gpurun_out/s3c_pytest.log)"
timeout 300 python scripts/tiled_phases.py 16777216 16384 64 > gpurun_out/s3_ph_cfg4d.txt 2>&1; echo "cfg4 ph rc $?"; tail -12 gpurun_out/s3_ph_cfg4d.txt
for w in cfg4 cfg4b; do
for i in 1 2 3; do
  for v in "" nocsm; do
    TM_LIB_VARIANT=$v timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
    echo "$w ${v:-new}: $(python scripts/show_bench.py gpurun_out/ab.log | cut -c1-150)"
  done
done
done
