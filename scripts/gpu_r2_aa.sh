mkdir -p gpurun_out
for w in cfg5 cfg4 cfg4a cfg4b cfg4c cfg4d; do bash scripts/gpu_ab_envvar.sh TM_FOLD_DUAL "0 1" 2 --workload $w; done
TM_FOLD_DUAL=1 timeout 900 python -m pytest "tests/test_fullsize_gpu.py::test_every_pair_int" "tests/test_parity_gpu.py::test_partial_folds_sum_to_full" "tests/test_parity_gpu.py::test_cfg5_full_size_fold_and_chunks" "tests/test_parity_gpu.py::test_packed_pm1_fold" "tests/test_multirank_gpu.py::test_fold_reduce_emulated_ranks" -q -x -p no:cacheprovider 2>&1 | tail -1
