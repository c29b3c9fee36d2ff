# Tensor-core correlation engine: parity tests first (bounded), then an A/B bench.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "tc_ or cfg1 or general_fold" > gpurun_out/pytest_tc.log 2>&1; echo pytest_tc rc=$?
tail -5 gpurun_out/pytest_tc.log
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_tc.log 2>&1; echo bench rc=$?
TM_CORR=ntt timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ntt.log 2>&1; echo bench_ntt rc=$?
python scripts/show_bench.py gpurun_out/bench_tc.log gpurun_out/bench_ntt.log 2>/dev/null || (tail -c 600 gpurun_out/bench_tc.log; tail -c 600 gpurun_out/bench_ntt.log)
