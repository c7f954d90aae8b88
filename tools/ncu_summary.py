#!/usr/bin/env python
"""Summarise one kernel of an ncu --set full report into the JSON bench.py reads.

    python tools/ncu_summary.py report.ncu-rep KERNEL_REGEX out.json "source description"
"""
import csv
import io
import json
import re
import subprocess
import sys

rep, kre, out, src = sys.argv[1:5]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, units = rows[0], rows[1]
kname = h.index("Kernel Name")
row = next(r for r in rows[2:] if re.search(kre, r[kname]))
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
m = {k: [row[h.index(k)], units[h.index(k)]] for k in want if k in h}


def nbytes(k):
    v, u = m[k]
    return float(v.replace(",", "")) * scale.get(u, 1)


rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
json.dump({"kernel": row[kname], "source": src, "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd,
           "dram_write_bytes": wr, "metrics": m}, open(out, "w"), indent=1)
print(json.dumps({"kernel": row[kname][:60], "us": m["gpu__time_duration.sum"], "dram_MB": (rd + wr) / 1e6}))
