mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_fullsize_gpu.py tests/test_multirank_gpu.py "tests/test_parity_gpu.py::test_partial_folds_sum_to_full" "tests/test_parity_gpu.py::test_packed_pm1_fold" "tests/test_parity_gpu.py::test_cfg5_full_size_fold_and_chunks" "tests/test_parity_gpu.py::test_randomized_large_shapes_sampled" "tests/test_parity_gpu.py::test_randomized_sweep_against_oracle" "tests/test_parity_gpu.py::test_back_to_back_staged_runs" -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu.log)"
for w in cfg5 cfg4 cfg4a cfg4b cfg4c; do
  for c in 0 1; do TM_FOLD_CONTIG=$c timeout 200 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/nt.log 2>&1; echo "$w contig=$c $(python scripts/show_bench.py gpurun_out/nt.log | cut -c1-170)"; done
done
