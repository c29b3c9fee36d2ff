timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_large_k_gpu.py tests/test_multirank_gpu.py tests/test_fullsize_gpu.py -k "tiled or tc_ or split or left or ragged or cfg5 or companions or ranks" -q -x -p no:cacheprovider > gpurun_out/pytest_red.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_red.log)"; grep -E "^FAILED" gpurun_out/pytest_red.log | head -3
bash scripts/gpu_ab_multi.sh "cur orig" 2 --workload cfg5 | cut -c1-125
C="python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tiled|match" -c 30 --csv --log-file gpurun_out/l_red.csv $C > gpurun_out/ncu.log 2>&1; echo "ncu rc $?"
python scripts/show_launches.py gpurun_out/l_red.csv 2>&1 | tail -3
