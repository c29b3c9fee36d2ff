# same-box A/B of an environment knob: bash scripts/gpu_ab_envvar.sh VAR "v1 v2" reps [bench args...]
mkdir -p gpurun_out
VAR=$1; VALS=$2; R=${3:-2}; shift 3
for i in $(seq $R); do
  for v in $VALS; do
    env $VAR=$v timeout 200 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 --no-cfg1 "$@" > gpurun_out/abv.log 2>&1
    echo "$i $VAR=$v $*: $(python scripts/show_bench.py gpurun_out/abv.log | cut -c9-150)"
  done
done
