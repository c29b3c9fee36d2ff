mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "ragged_last_block" 2>&1 | tail -3
timeout 420 python scripts/sweep_many.py 0 4000 > gpurun_out/sweep_many.log 2>&1; echo "many rc $? $(tail -1 gpurun_out/sweep_many.log)"
timeout 400 python scripts/sweep_wide.py 0 1200 > gpurun_out/sweep_wide.log 2>&1; echo "wide rc $? $(tail -1 gpurun_out/sweep_wide.log)"
timeout 300 python scripts/sweep_extra.py 300 > gpurun_out/sweep_extra.log 2>&1; echo "extra rc $? $(tail -1 gpurun_out/sweep_extra.log)"
grep FAIL gpurun_out/sweep_wide.log | head -5 | cut -c1-300
grep FAIL gpurun_out/sweep_extra.log | head -5 | cut -c1-300
