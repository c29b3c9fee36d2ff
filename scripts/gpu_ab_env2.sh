# same-box A/B of an environment switch: bash scripts/gpu_ab_env2.sh "ENV=1" [reps] [bench args...]
mkdir -p gpurun_out
E=$1; R=${2:-3}; shift 2
for i in $(seq $R); do
  timeout 120 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 "$@" > gpurun_out/ab_base.log 2>&1
  env $E timeout 120 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 "$@" > gpurun_out/ab_var.log 2>&1
  echo "base: $(python scripts/show_bench.py gpurun_out/ab_base.log | cut -c10-38)   $E: $(python scripts/show_bench.py gpurun_out/ab_var.log | cut -c9-37)"
done
