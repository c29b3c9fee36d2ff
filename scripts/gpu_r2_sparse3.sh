mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -k "tiled_sparse or tc_one_cta_and_tiled or tc_engine_limbs" -q -x -p no:cacheprovider > gpurun_out/pytest_sparse.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_sparse.log)"
TM_LIB_VARIANT=pc timeout 900 python -m pytest tests/test_parity_gpu.py -k "tiled_sparse" -q -x -p no:cacheprovider > gpurun_out/pytest_sparse_pc.log 2>&1; echo "tests pc: $(tail -1 gpurun_out/pytest_sparse_pc.log)"
bash scripts/gpu_ab_multi.sh "base pc m2 m4" 2 --workload cfg4
bash scripts/gpu_ab_multi.sh "base m2 m4" 1 --workload cfg5
for sp in 1 0; do echo "phases sparse=$sp"; TM_TILED_SPARSE=$sp timeout 300 python scripts/tiled_phases.py 16777216 16384 64 2>&1 | tail -9 | head -5; done
echo "phases pc"; TM_LIB_VARIANT=pc timeout 300 python scripts/tiled_phases.py 16777216 16384 64 2>&1 | tail -9 | head -5
C="python bench.py --workload cfg4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
$C > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tiled|fold" -c 40 --csv --log-file gpurun_out/launches_cfg4.csv $C > gpurun_out/ncu.log 2>&1; echo "ncu rc $?"
python scripts/show_launches.py gpurun_out/launches_cfg4.csv 2>&1 | tail -6
