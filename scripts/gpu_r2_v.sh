mkdir -p gpurun_out
for v in base cores; do for c in 1 2 4; do
  if [ $v = base ]; then timeout 120 python scripts/overlap_probe.py 16777216 16384 64 $c; else TM_LIB_VARIANT=cores timeout 120 python scripts/overlap_probe.py 16777216 16384 64 $c; fi
done; done
TM_LIB_VARIANT=cores timeout 120 python scripts/overlap_probe.py 16777216 32768 64 4
timeout 120 python scripts/overlap_probe.py 16777216 32768 64 1
