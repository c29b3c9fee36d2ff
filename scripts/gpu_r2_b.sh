# round 2, call b: large-K parity, K transition, cfg4 companions, ncu of the cfg5 kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_large_k_gpu.py "tests/test_fullsize_gpu.py::test_general_int8_all_limbs" -q --timeout 1200 -p no:cacheprovider --durations=10 > gpurun_out/pytest_largek.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_largek.log)"
timeout 900 python scripts/k_transition.py 12 64 > gpurun_out/k_transition.json 2> gpurun_out/k_transition.err; echo "ktrans rc $?"
for w in cfg4c cfg4d; do timeout 300 python bench.py --workload $w --no-cpu-baseline --no-cfg1 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc $?"; done
C="python bench.py --workload cfg5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
$C > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"corr_tc_tiled|fold_pm1_tma|fold_finalize" -s 6 -c 3 -o gpurun_out/prof_cfg5 $C > gpurun_out/ncu_cfg5.log 2>&1; echo "ncu rc $?"
$C > gpurun_out/plain2.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/launches_cfg5.csv $C > /dev/null 2>&1; echo "ncu2 rc $?"
