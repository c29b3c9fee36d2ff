for i in 1 2; do
for cfg in "0 0" "32 9" "64 18" "64 9" "64 12"; do set -- $cfg
  if [ $1 = 0 ]; then unset TM_TILED_NT TM_TILED_NCR; else export TM_TILED_NT=$1 TM_TILED_NCR=$2; fi
  timeout 200 python bench.py --workload cfg5 --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "$i cfg5 nt=$1 ncr=$2 $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-110)"
done; done
