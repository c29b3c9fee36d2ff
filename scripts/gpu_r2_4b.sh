for i in 1 2; do for w in cfg4b cfg4a; do for tl in default 1; do
  if [ $tl = 1 ]; then export TM_TC_TILED=1; else unset TM_TC_TILED; fi
  timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "$i $w tiled=$tl $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-130)"
done; done; done
unset TM_TC_TILED
echo phases-4b; TM_TC_TILED=1 timeout 300 python scripts/tiled_phases.py 16777216 8192 64 2>&1 | tail -10
