# same-box A/B of an env switch on the default bench: bash scripts/gpu_ab_env.sh VAR=VAL [reps]
mkdir -p gpurun_out
for i in $(seq ${2:-3}); do
  timeout 120 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab_base.log 2>&1
  env $1 timeout 120 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab_var.log 2>&1
  echo "base: $(python scripts/show_bench.py gpurun_out/ab_base.log | cut -c1-40)   $1: $(python scripts/show_bench.py gpurun_out/ab_var.log | cut -c1-40)"
done
