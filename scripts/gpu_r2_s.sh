mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu.log)"
timeout 600 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "cfg5 $(python scripts/show_bench.py gpurun_out/bench_cfg5.json | cut -c1-200)"
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $? $(cut -c1-300 gpurun_out/bench_ref.json)"
