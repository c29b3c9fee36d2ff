# bench every workload once (short), default engine and NTT engine
mkdir -p gpurun_out
for w in cfg1 cfg3 cfg4a cfg4b cfg4 cfg5; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bw_$w.log 2>&1; echo "$w rc=$?"
  TM_CORR=ntt timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bw_${w}_ntt.log 2>&1
done
for f in gpurun_out/bw_*.log; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f.split('/')[-1], round(d['value'], 1), 'ms', round(d['ms_per_step'], 4), d.get('run_path', ''), {k: round(v, 4) for k, v in d.get('stage_ms', {}).items()}, 'frac', round(d['roofline']['frac'], 3))
except Exception as e:
    print(f, 'ERR', e, open(f).read()[-300:])
PY
done
