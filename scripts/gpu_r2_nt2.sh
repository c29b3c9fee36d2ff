for w in cfg4 cfg4c; do
for cfg in "0 0" "64 1" "64 2" "32 2"; do set -- $cfg
  if [ $1 = 0 ]; then unset TM_TILED_NT TM_TILED_NCR; else export TM_TILED_NT=$1 TM_TILED_NCR=$2; fi
  timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "$w nt=$1 ncr=$2 $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-130)"
done; done
unset TM_TILED_NT TM_TILED_NCR
for w in cfg4a cfg4b; do for tl in default 1; do
  if [ $tl = 1 ]; then export TM_TC_TILED=1; else unset TM_TC_TILED; fi
  timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "$w tiled=$tl $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-130)"
done; done
