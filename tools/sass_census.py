"""SASS instruction census of libfvsr_b200.so per kernel (Blackwell-native evidence):
tcgen05 MMA (UTCHMMA), TMEM loads/stores (LDTM/STTM), TMEM alloc (UTCATOM*/UTC*),
bulk copies (UBLKCP), tensor-map TMA (UTMALDG), mbarrier ops (SYNCS), MUFU.EX2, FMUL2/FADD2.

    python tools/sass_census.py [lib.so] [out.json]
"""
import collections
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "..", "paper_2510_12747_b200", "libfvsr_b200.so")
out = sys.argv[2] if len(sys.argv) > 2 else None
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
KEYS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTCATOMSWS", "UBLKCP", "UBLKPF", "UTMALDG", "UTMASTG", "SYNCS",
        "MUFU.EX2", "FMUL2", "FADD2", "FFMA2", "F2FP", "VOTE", "POPC", "REDG", "ATOMG", "BAR"]
census = {}
fn = None
counts = collections.Counter()
for line in txt.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        if fn:
            census[fn] = dict(counts)
        fn, counts = m.group(1), collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if m and fn:
        op = m.group(2)
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                counts[k] += 1
        counts["_total"] += 1
if fn:
    census[fn] = dict(counts)


def short(name):
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    return d.split("(")[0].replace("void ", "")


res = {short(k): v for k, v in sorted(census.items())}
doc = {"library": os.path.basename(lib), "tool": "cuobjdump -sass | tools/sass_census.py", "kernels": res}
if out:
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
for k, v in res.items():
    interesting = {kk: vv for kk, vv in v.items() if kk in ("UTCHMMA", "LDTM", "STTM", "UBLKCP", "UTMALDG", "MUFU.EX2",
                                                            "FMUL2", "FADD2", "SYNCS", "_total")}
    print(f"{k[:60]:60s} {interesting}")
