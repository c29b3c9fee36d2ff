mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_large_k_gpu.py "tests/test_parity_gpu.py::test_tc_one_cta_and_tiled_kernels" "tests/test_parity_gpu.py::test_split_correlation_parts_max_equals_whole" "tests/test_fullsize_gpu.py::test_every_pair_int" "tests/test_fullsize_gpu.py::test_cfg5_whole_signal_equals_oracle" "tests/test_parity_gpu.py::test_f32_small" "tests/test_parity_gpu.py::test_cfg3_full_batch_sampled" -q --timeout 900 -p no:cacheprovider --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu.log)"
for w in cfg5 cfg4 cfg4c cfg4d; do
  for nt in 32 64; do TM_TILED_NT=$nt timeout 200 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/nt.log 2>&1; echo "$w NT=$nt $(python scripts/show_bench.py gpurun_out/nt.log | cut -c1-150)"; done
done
TRIALS=40 timeout 300 python scripts/table2.py > gpurun_out/table2.txt 2>&1; tail -2 gpurun_out/table2.txt
timeout 200 python bench.py --workload t2 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/t2.log 2>&1; echo "t2 $(python scripts/show_bench.py gpurun_out/t2.log | cut -c1-200)"
C="python bench.py --workload cfg5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
$C > gpurun_out/plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches_cfg5.csv $C > /dev/null 2>&1; echo "ncu rc $?"
