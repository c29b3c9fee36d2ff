import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split('/')[-1], round(d['value'], 1), 'ms/step', round(d['ms_per_step'], 4),
              {k: round(v, 4) for k, v in d['stage_ms'].items()}, 'frac', round(d['roofline']['frac'], 3),
              'clk', d.get('clocks', {}).get('sm_mhz'), d.get('run_path', '')[:24])
    except Exception as e:
        print(f, 'ERR', e)
