for cfg in "32 0" "64 1" "64 2"; do set -- $cfg
  TM_TILED_NT=$1 TM_TILED_NCR=$2 timeout 200 python bench.py --workload cfg4 --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "nt=$1 ncr=$2 $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-130)"
  echo "phases"; TM_TILED_NT=$1 TM_TILED_NCR=$2 timeout 300 python scripts/tiled_phases.py 16777216 16384 64 2>&1 | tail -8
done
