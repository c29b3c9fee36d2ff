for i in 1 2; do for w in cfg4a cfg4 cfg4b; do for f in 0 1; do
  TM_FIN_BINS=$f timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 > gpurun_out/ab.log 2>&1
  echo "$i $w fin=$f $(python scripts/show_bench.py gpurun_out/ab.log | cut -c9-110)"
done; done; done
