import csv, sys
from collections import defaultdict
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[hi]; idx={k:i for i,k in enumerate(h)}
agg=defaultdict(list)
for r in rows[hi+1:]:
    if len(r)<len(h) or r[idx['Metric Name']]!='gpu__time_duration.sum': continue
    agg[r[idx['Kernel Name']].split('(')[0][:50]].append(float(r[idx['Metric Value']]))
tot=sum(sum(v) for v in agg.values())
for k,v in sorted(agg.items(), key=lambda kv:-sum(kv[1])):
    print(f"{k:50s} n={len(v):4d} mean={sum(v)/len(v)/1e3:9.2f}us share={sum(v)/tot*100:5.1f}%")
