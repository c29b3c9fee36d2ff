# same-box A/B of several library variants: bash scripts/gpu_ab_multi.sh "base nst5 ..." reps [bench args...]
mkdir -p gpurun_out
VARS=$1; R=${2:-3}; shift 2
for i in $(seq $R); do
  for v in $VARS; do
    if [ "$v" = base ] || [ "$v" = cur ]; then
      timeout 200 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 "$@" > gpurun_out/ab_$v.log 2>&1
    else
      TM_LIB_VARIANT=$v timeout 200 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 "$@" > gpurun_out/ab_$v.log 2>&1
    fi
    echo "$i $v: $(python scripts/show_bench.py gpurun_out/ab_$v.log | cut -c1-160)"
  done
done
