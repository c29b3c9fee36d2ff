# like gpu_ab_var.sh but the variant is the OLD build: prints base (current) vs old
mkdir -p gpurun_out
V=$1; R=${2:-3}; shift 2
for i in $(seq $R); do
  timeout 120 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 "$@" > gpurun_out/ab_base.log 2>&1
  TM_LIB_VARIANT=$V timeout 120 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 "$@" > gpurun_out/ab_var.log 2>&1
  echo "new: $(python scripts/show_bench.py gpurun_out/ab_base.log | cut -c10-38)   $V: $(python scripts/show_bench.py gpurun_out/ab_var.log | cut -c9-37)"
done
