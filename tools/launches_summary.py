import csv, sys
from collections import defaultdict
rows=list(csv.reader(open(sys.argv[1])))
hdr=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
agg=defaultdict(list)
for r in rows[hdr+1:]:
    if len(r)>vi: agg[r[ki][:70]].append(float(r[vi].replace(',','')))
tot=sum(sum(v)/len(v) for v in agg.values())
for k,v in agg.items(): print(f"{k:70s} n={len(v):3d} mean={sum(v)/len(v)/1e3:10.1f} us  share={sum(v)/len(v)/tot:6.1%}")
