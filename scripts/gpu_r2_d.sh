mkdir -p gpurun_out
timeout 300 python scripts/pattern_probe.py > gpurun_out/pattern_probe.json 2> gpurun_out/pattern_probe.err; echo "probe rc $?"; cat gpurun_out/pattern_probe.json
timeout 300 python scripts/tiled_phases.py 2147483648 65536 1 > gpurun_out/tiled_cfg5.txt 2>&1; echo "phases5 rc $?"; cat gpurun_out/tiled_cfg5.txt
timeout 300 python scripts/tiled_phases.py 16777216 16384 64 > gpurun_out/tiled_cfg4.txt 2>&1; echo "phases4 rc $?"; cat gpurun_out/tiled_cfg4.txt
timeout 900 python -m pytest tests/test_large_k_gpu.py::test_plan_beyond_ntt_tables -q -p no:cacheprovider 2>&1 | tail -2
