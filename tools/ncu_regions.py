#!/usr/bin/env python
"""Per-region warp-stall samples of the attention kernel from an ncu source page (SASS csv).

    ncu -i X.ncu-rep --page source --csv --print-source sass > src.csv
    python tools/ncu_regions.py src.csv [top]
Regions: setup | producer/issuer/epilogue warpgroup (after setmaxnreg.dec) | softmax (after
setmaxnreg.inc).  Prints sample totals with the stall breakdown and the top instructions.
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith('stall_') and 'Not Issued' not in k]
body = rows[2:]
region = 'setup'
agg = {}
inst = []
for i, r in enumerate(body):
    src = r[ix['Source']]
    if 'USETMAXREG.DEALLOC' in src:
        region = 'other'
    elif 'USETMAXREG.TRY_ALLOC' in src:
        region = 'softmax'
    s = int(r[ix['Warp Stall Sampling (All Samples)']] or 0)
    a = agg.setdefault(region, {'samples': 0, 'inst': 0, **{k: 0 for k in stalls}})
    a['samples'] += s
    a['inst'] += int(r[ix['Instructions Executed']] or 0)
    for k in stalls:
        a[k] += int(r[ix[k]] or 0)
    inst.append((s, i, region, src.strip(), {k: int(r[ix[k]] or 0) for k in stalls}))
tot = sum(a['samples'] for a in agg.values())
for reg, a in agg.items():
    br = sorted(((a[k], k) for k in stalls), reverse=True)[:6]
    print(f"{reg:8s} samples {a['samples']:7d} ({100*a['samples']/tot:4.1f}%) warp-inst {a['inst']:9d}  " +
          ' '.join(f"{k[6:]}={v}" for v, k in br))
print()
for s, i, reg, src, st in sorted(inst, reverse=True)[:top]:
    br = sorted(((v, k) for k, v in st.items()), reverse=True)[:3]
    print(f"{s:6d} {i:5d} {reg:7s} {src[:60]:60s} " + ' '.join(f"{k[6:]}={v}" for v, k in br))
