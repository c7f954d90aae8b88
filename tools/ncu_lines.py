"""Top source lines by warp-stall samples from an ncu report (cuda,sass source page).

    python tools/ncu_lines.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
fname = ""
out = []
hdr = None
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 6 or not r[0]:
        continue
    try:
        w = int(r[4] or 0)
        e = int(r[7] or 0)
    except ValueError:
        continue
    out.append((w, fname, r[0], e, r[1].strip()[:100]))
tot = sum(o[0] for o in out) or 1
out.sort(reverse=True)
for w, f, ln, e, s in out[:top]:
    print("%5.1f%% %18s:%-5s %9d  %s" % (100.0 * w / tot, f, ln, e, s))
