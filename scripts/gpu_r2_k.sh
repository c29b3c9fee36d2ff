mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_large_k_gpu.py tests/test_fullsize_gpu.py tests/test_multirank_gpu.py "tests/test_parity_gpu.py::test_tc_one_cta_and_tiled_kernels" "tests/test_parity_gpu.py::test_split_correlation_parts_max_equals_whole" "tests/test_parity_gpu.py::test_back_to_back_staged_runs" "tests/test_parity_gpu.py::test_randomized_large_shapes_sampled" -q -x --timeout 900 -p no:cacheprovider -s > gpurun_out/pytest_gpu.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu.log)"; grep "fused combine paths" gpurun_out/pytest_gpu.log
for w in cfg5 cfg4 cfg4c; do timeout 200 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/nt.log 2>&1; echo "$w $(python scripts/show_bench.py gpurun_out/nt.log | cut -c1-150)"; done
C="python bench.py --workload cfg5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
$C > gpurun_out/plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 24 --csv --log-file gpurun_out/launches_cfg5.csv $C > /dev/null 2>&1; echo "ncu rc $?"
