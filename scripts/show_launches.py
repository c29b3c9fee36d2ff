import csv, sys
from collections import defaultdict
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hdr]
    ki, mi, vi, ui, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit'), h.index('ID')
    agg = defaultdict(lambda: defaultdict(list))
    for r in rows[hdr + 1:]:
        if len(r) <= vi: continue
        v = float(r[vi].replace(',', ''))
        u = r[ui]
        if u == 'nsecond': v /= 1e3
        elif u == 'usecond': pass
        elif u == 'msecond': v *= 1e3
        elif u in ('byte',): v /= 1e6
        elif u == 'Kbyte': v /= 1e3
        elif u == 'Gbyte': v *= 1e3
        agg[r[ki][:50]][r[mi]].append(v)
    print(f)
    for k, m in agg.items():
        t = m.get('gpu__time_duration.sum', [0]); rd = m.get('dram__bytes_read.sum', [0]); wr = m.get('dram__bytes_write.sum', [0])
        print(f"  {k:50s} n={len(t):3d} t={sum(t)/len(t):8.1f}us  read={sum(rd)/len(rd):8.2f}MB write={sum(wr)/len(wr):8.2f}MB")
