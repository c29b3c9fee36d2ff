timeout 900 python -m pytest tests/test_parity_gpu.py -k "tiled" -q -x -p no:cacheprovider > gpurun_out/pytest_gw.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gw.log)"
for w in cfg4 cfg5; do bash scripts/gpu_ab_multi.sh "cur gw0 sus" 1 --workload $w | cut -c1-125; done
for v in cur gw0; do echo "phases $v"; if [ $v = gw0 ]; then export TM_LIB_VARIANT=gw0; fi; timeout 300 python scripts/tiled_phases.py 16777216 16384 64 2>&1 | tail -9; done
