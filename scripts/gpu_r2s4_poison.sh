mkdir -p gpurun_out
if [ -f paper_1509_04863_b200/libtm_7e0d04d.so ]; then echo "pre-fix library, split tests (must fail): $(TM_LIB_VARIANT=7e0d04d timeout 300 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k split_correlation 2>&1 | tail -1)"; fi
echo "final library, split tests: $(timeout 300 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k split_correlation 2>&1 | tail -1)"
TM_WS_POISON=0xFF timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu_poison_ff.log 2>&1; echo "suite, workspaces 0xFF: $(tail -1 gpurun_out/pytest_gpu_poison_ff.log)"
grep -E "^FAILED|^ERROR" gpurun_out/pytest_gpu_poison_ff.log | head -20
TM_WS_POISON=0xFF timeout 300 python scripts/sweep_many.py 0 1500 > gpurun_out/sweep_many_p.log 2>&1; echo "many 0xFF rc $? $(tail -1 gpurun_out/sweep_many_p.log)"
TM_WS_POISON=0xFF timeout 300 python scripts/sweep_wide.py 0 500 > gpurun_out/sweep_wide_p.log 2>&1; echo "wide 0xFF rc $? $(tail -1 gpurun_out/sweep_wide_p.log)"
TM_WS_POISON=0xFF timeout 200 python scripts/sweep_extra.py 200 > gpurun_out/sweep_extra_p.log 2>&1; echo "extra 0xFF rc $? $(tail -1 gpurun_out/sweep_extra_p.log)"
