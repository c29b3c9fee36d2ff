mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_parity_gpu.py tests/test_abi.py -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu.log)"
python -c "import __graft_entry__ as g; g.smoke()"
timeout 200 python bench.py --workload cfg1 --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c1.log 2>&1; tail -c 600 gpurun_out/c1.log
TM_SMALL=0 timeout 200 python bench.py --workload cfg2 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c2.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/c2.log').read().strip().splitlines()[-1]); print('cfg1 staged', d['cfg1_latency'])"
