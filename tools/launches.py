import csv, sys
from collections import defaultdict
rows=list(csv.reader(open(sys.argv[1])))
hdr=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=defaultdict(lambda:[0,0.0]); tot=0.0
for r in rows[hdr+1:]:
    if len(r)>vi:
        try: v=float(r[vi].replace(',',''))
        except: continue
        agg[r[ki][:70]][0]+=1; agg[r[ki][:70]][1]+=v; tot+=v
for k,(n,t) in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{t/1e3:10.1f} us total {n:4d} launches {t/1e3/n:9.1f} us/launch {100*t/tot:5.1f}%  {k}")
