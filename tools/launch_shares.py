import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None;agg=collections.defaultdict(lambda:[0,0.0])
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get('Metric Name')=='gpu__time_duration.sum':
            k=d['Kernel Name'][:80]; agg[k][0]+=1; agg[k][1]+=float(d['Metric Value'].replace(',',''))
tot=sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(),key=lambda x:-x[1][1]): print(f"{v[1]/1e3:10.1f} us {v[0]:4d}x {100*v[1]/tot:5.1f}%  {k}")
