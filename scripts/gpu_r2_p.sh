mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_fullsize_gpu.py "tests/test_parity_gpu.py::test_partial_folds_sum_to_full" "tests/test_parity_gpu.py::test_packed_pm1_fold" "tests/test_parity_gpu.py::test_packed_pm1_extremes" "tests/test_parity_gpu.py::test_cfg5_full_size_fold_and_chunks" "tests/test_parity_gpu.py::test_randomized_large_shapes_sampled" "tests/test_parity_gpu.py::test_randomized_sweep_against_oracle" -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu.log)"
for w in cfg5 cfg4 cfg4a cfg4b; do bash scripts/gpu_ab_multi.sh "base late" 1 --workload $w; done
bash scripts/gpu_ab_multi.sh "base late" 1 --workload cfg5
