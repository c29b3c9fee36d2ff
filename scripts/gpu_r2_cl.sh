mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_large_k_gpu.py tests/test_multirank_gpu.py -k "tiled or tc_ or split or left or ragged or cfg5 or companions or ranks or many" -q -x -p no:cacheprovider > gpurun_out/pytest_cl.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_cl.log)"
grep -E "^FAILED|Error" gpurun_out/pytest_cl.log | head -5
for i in 1 2; do for cl in 1 0; do
  TM_DEBUG_CL=1 TM_TILED_CL=$cl timeout 200 python bench.py --workload cfg5 --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "$i cl=$cl $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-120)"; grep "tm: cluster" gpurun_out/ab.log | sort | uniq | head -4
done; done
timeout 300 python scripts/tiled_phases.py 2147483648 65536 1 2>&1 | tail -9 | head -6
C="python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tiled|match" -c 30 --csv --log-file gpurun_out/l_cl.csv $C > gpurun_out/ncu.log 2>&1; echo "ncu rc $?"
python scripts/show_launches.py gpurun_out/l_cl.csv 2>&1 | tail -3
