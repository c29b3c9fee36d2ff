# sparse single-limb tiled correlation: parity + cfg4 A/B (sparse on/off, NT 32/64)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -k "tiled_sparse or tc_one_cta_and_tiled or tc_engine_limbs" -q -x -p no:cacheprovider > gpurun_out/pytest_sparse.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_sparse.log)"
timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1; echo "full: $(tail -1 gpurun_out/pytest_full.log)"
for i in 1 2; do
for sp in 1 0; do for nt in 32 64; do
  TM_TILED_SPARSE=$sp TM_TILED_NT=$nt timeout 200 python bench.py --workload cfg4 --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "$i sparse=$sp nt=$nt $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-150)"
done; done; done
for w in cfg4b cfg5; do
  timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "$w $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-150)"
done
