for i in 1 2 3; do for w in cfg4a cfg4b; do for fw in 1 0; do
  TM_FIN_WHOLE=$fw timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "$i $w fw=$fw $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-120)"
done; done; done
