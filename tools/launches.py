"""Summarise an ncu launch list (gpu__time_duration.sum per launch).

    python tools/launches.py launches.csv [--skip N]

--skip drops the first N launches (e.g. the ring prefill appends before the timed steps).
Per-launch times are cold-cache and serialised: compare shares, not absolutes."""
import csv
import sys
from collections import defaultdict

args = sys.argv[1:]
skip = 0
if "--skip" in args:
    i = args.index("--skip")
    skip = int(args[i + 1])
    del args[i:i + 2]
rows = list(csv.reader(open(args[0])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
idx = {k: i for i, k in enumerate(h)}
launches = [r for r in rows[hi + 1:] if len(r) >= len(h) and r[idx["Metric Name"]] == "gpu__time_duration.sum"]
agg = defaultdict(list)
for r in launches[skip:]:
    agg[r[idx["Kernel Name"]].split("(")[0][:50]].append(float(r[idx["Metric Value"]]))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:50s} n={len(v):4d} mean={sum(v)/len(v)/1e3:9.2f}us share={sum(v)/tot*100:5.1f}%")
