# A/B of the tensor-core overlap mode (fold of chunk c+1 || correlation of chunk c)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "cfg2 or cfg1 or tc_" > gpurun_out/pytest_ovl.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_ovl.log
for ch in 4 8 12 16; do
TM_OVERLAP_CHUNKS=$ch timeout 120 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ovl$ch.log 2>&1; echo ovl$ch rc=$?
done
TM_OVERLAP=0 timeout 120 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_noovl.log 2>&1
python scripts/show_bench.py gpurun_out/bench_ovl*.log gpurun_out/bench_noovl.log
