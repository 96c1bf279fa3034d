import csv, collections, sys
lines=[l for l in open(sys.argv[1]) if l.startswith('"')]
rows=list(csv.reader(lines))
hdr=rows[0]
i_name=hdr.index('Kernel Name'); i_val=hdr.index('Metric Value'); i_grid=hdr.index('Grid Size')
tot=collections.defaultdict(float); cnt=collections.Counter()
seq=[]
for r in rows[1:]:
    try: v=float(r[i_val].replace(',',''))
    except: continue
    n=r[i_name].split('(')[0]
    if n.startswith('void '): n=n[5:]
    n=n.split('<')[0]
    tot[n]+=v; cnt[n]+=1; seq.append((n, v, r[i_grid]))
T=sum(tot.values())
for n,v in sorted(tot.items(), key=lambda x:-x[1]):
    print(f"{n:40s} {cnt[n]:5d} {v/1e3:10.1f} us  {100*v/T:5.1f}%  avg {v/cnt[n]/1e3:.2f} us")
print("total us", T/1e3, "launches", sum(cnt.values()))
if len(sys.argv)>2:
    for n,v,g in seq[:int(sys.argv[2])]: print(f"  {n:30s} {g:15s} {v/1e3:8.2f}")
