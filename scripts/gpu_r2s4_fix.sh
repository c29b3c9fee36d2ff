mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "split_correlation or ragged_last_block" 2>&1 | tail -3
timeout 300 python scripts/sweep_extra.py 400 > gpurun_out/sweep_extra.log 2>&1; echo "extra rc $? $(tail -1 gpurun_out/sweep_extra.log)"
grep FAIL gpurun_out/sweep_extra.log | head -5 | cut -c1-300
