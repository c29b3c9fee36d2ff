import re,csv,collections,sys
sassf, csvf, fn = sys.argv[1], sys.argv[2], sys.argv[3]
lines=open(sassf).read().split('\n')
st=[i for i,l in enumerate(lines) if l.startswith('.text.') and fn in l][0]
cur=None; addr2line={}
for l in lines[st+1:]:
    if l.startswith('.text.'): break
    m=re.search(r'//## File "([^"]+)", line (\d+)',l)
    if m: cur=(m.group(1).split('/')[-1],int(m.group(2)))
    m=re.match(r'\s+/\*([0-9a-f]{4,})\*/',l)
    if m: addr2line[int(m.group(1),16)]=cur
rows=list(csv.reader(open(csvf)))
h=rows[1]; ai=h.index('Address'); ie=h.index('Instructions Executed'); si=h.index('Warp Stall Sampling (All Samples)')
base=None; agg=collections.Counter(); st_=collections.Counter()
for r in rows[2:]:
    try: a=int(r[ai],16)
    except: continue
    if base is None: base=a
    ln=addr2line.get(a-base)
    agg[ln]+=float(r[ie] or 0); st_[ln]+=float(r[si] or 0)
tot=sum(agg.values()); tots=sum(st_.values())
print('total warp inst',tot,'samples',tots)
for ln,v in sorted(agg.items(),key=lambda x:-x[1])[:int(sys.argv[4]) if len(sys.argv)>4 else 30]:
    print(ln, f'{v/tot*100:5.1f}% inst  {st_[ln]/tots*100:5.1f}% stall')
