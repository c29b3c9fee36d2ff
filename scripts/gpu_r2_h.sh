mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_large_k_gpu.py tests/test_fullsize_gpu.py tests/test_multirank_gpu.py "tests/test_parity_gpu.py::test_tc_one_cta_and_tiled_kernels" "tests/test_parity_gpu.py::test_split_correlation_parts_max_equals_whole" "tests/test_parity_gpu.py::test_back_to_back_staged_runs" -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu.log)"
for w in cfg5 cfg4 cfg4b cfg4c cfg4d; do
  for nt in 32 64; do TM_TILED_NT=$nt timeout 200 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/nt.log 2>&1; echo "$w NT=$nt $(python scripts/show_bench.py gpurun_out/nt.log | cut -c1-150)"; done
  TM_LIB_VARIANT=old_tiled timeout 200 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/nt.log 2>&1; echo "$w old $(python scripts/show_bench.py gpurun_out/nt.log | cut -c1-150)"
done
TM_TC_TILED=1 timeout 200 python bench.py --workload cfg4b --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/t.log 2>&1; echo "cfg4b tiled64 $(python scripts/show_bench.py gpurun_out/t.log | cut -c1-150)"
TM_TC_TILED=1 timeout 200 python bench.py --workload cfg4a --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/t.log 2>&1; echo "cfg4a tiled64 $(python scripts/show_bench.py gpurun_out/t.log | cut -c1-150)"
C="python bench.py --workload cfg5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
$C > gpurun_out/plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg5.csv $C > /dev/null 2>&1; echo "ncu rc $?"
