"""Aggregate ncu warp-stall samples (--page source --print-source sass --csv) by
CUDA source line, using the -lineinfo of the cubin (nvdisasm -g).
usage: python scripts/ncu_lines.py sass.csv kernel.cubin kernel_substring source.cu [n]"""
import csv, re, subprocess, sys

sass_csv, cubin, kname, srcfile = sys.argv[1:5]
n = int(sys.argv[5]) if len(sys.argv) > 5 else 25
out = subprocess.run(['nvdisasm', '-g', cubin], capture_output=True, text=True).stdout.split('\n')
amap, cur, on = {}, None, False
for l in out:
    if l.lstrip().startswith('.section'):
        on = ('.text.' in l) and (kname in l)
        continue
    if not on:
        continue
    m = re.search(r'//## File "(.*?)", line (\d+)', l)
    if m:
        cur = int(m.group(2)) if m.group(1).endswith(srcfile.split('/')[-1]) else -1
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4})\*/', l)
    if m:
        amap[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
hdr, data = rows[1], rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not' not in h]
base = int(data[0][0], 16)
agg, why = {}, {}
for r in data:
    ln = amap.get(int(r[0], 16) - base)
    v = int(r[iS]) if r[iS].isdigit() else 0
    agg[ln] = agg.get(ln, 0) + v
    w = why.setdefault(ln, {})
    for i, h in stall_cols:
        if r[i].isdigit() and int(r[i]):
            w[h] = w.get(h, 0) + int(r[i])
src = open(srcfile).read().split('\n')
tot = sum(agg.values()) or 1
for ln, v in sorted(agg.items(), key=lambda x: -x[1])[:n]:
    top = sorted(why[ln].items(), key=lambda x: -x[1])[:3]
    print(f'{v:6d} {100 * v / tot:5.1f}%  L{ln}: {src[ln - 1].strip()[:70] if ln and ln > 0 else 'other file'}  {top}')
