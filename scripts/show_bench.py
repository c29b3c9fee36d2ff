import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).readline())
        print(f.split('/')[-1], round(d['value'], 1), 'ms/step', round(d['ms_per_step'], 4),
              {k: round(v, 4) for k, v in d['stage_ms'].items()}, 'fold frac', round(d["roofline"]["frac"], 3), d.get("run_path", "")[:20])
    except Exception as e:
        print(f, 'ERR', e)
