mkdir -p gpurun_out
for w in cfg5 cfg4 cfg4a cfg4b; do bash scripts/gpu_ab_multi.sh "base two twob" 1 --workload $w; done
TM_LIB_VARIANT=two timeout 900 python -m pytest "tests/test_fullsize_gpu.py::test_every_pair_int" "tests/test_parity_gpu.py::test_partial_folds_sum_to_full" "tests/test_parity_gpu.py::test_cfg5_full_size_fold_and_chunks" -q -x -p no:cacheprovider 2>&1 | tail -1
