mkdir -p gpurun_out
bash scripts/gpu_ab_multi.sh "base pre" 3 --workload cfg2
timeout 1800 python -m pytest tests/test_multirank_gpu.py "tests/test_parity_gpu.py::test_split_correlation_parts_max_equals_whole" "tests/test_parity_gpu.py::test_tc_one_cta_and_tiled_kernels" tests/test_large_k_gpu.py -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu.log)"
