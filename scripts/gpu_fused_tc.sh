# fused fold + tensor-core correlation kernel: parity (bounded), then A/B bench
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "cfg2 or cfg1 or tc_ or packed" > gpurun_out/pytest_ftc.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_ftc.log
timeout 120 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ftc.log 2>&1; echo ftc rc=$?
TM_FUSED_TC=0 timeout 120 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_noftc.log 2>&1
python scripts/show_bench.py gpurun_out/bench_ftc.log gpurun_out/bench_noftc.log
