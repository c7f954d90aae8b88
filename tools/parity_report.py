"""Per-shape parity table from the GPU suite's record_parity lines.

    FVSR_PARITY_REPORT=gpurun_out/parity.jsonl python -m pytest tests -m gpu
    python tools/parity_report.py gpurun_out/parity.jsonl profiles/parity_r2.json

Writes {"cases": [...], "tolerance": {...}} and prints a markdown table (BASELINE.md's
"GPU results" table is this table).
"""
import json
import sys


def main(src, dst):
    cases = {}
    for line in open(src):
        line = line.strip()
        if line:
            r = json.loads(line)
            cases[r["case"]] = r  # last run of a case wins
    from tests.helpers import MAX_ABS_TOL, REL_L2_TOL
    out = {"tolerance": {"rel_l2": REL_L2_TOL, "max_abs": MAX_ABS_TOL},
           "indices": "bit-exact (selected ids, counts, diagonal; coarse-score bits where compared)",
           "cases": list(cases.values())}
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print("| case | shape | heads | k | indices | rel-L2 | max-abs |")
    print("|---|---|---|---|---|---|---|")
    for r in cases.values():
        shape = "%sx%s" % (r.get("rows", "?"), r.get("cols", "?"))
        rl = "%.2e" % r["rel_l2"] if "rel_l2" in r else "—"
        ma = "%.2e" % r["max_abs"] if "max_abs" in r else "—"
        print("| %s | %s | %s | %s | %s | %s | %s |" % (r["case"], shape, r.get("heads", "?"), r.get("topk", "?"),
                                                      "exact" if r.get("indices_bit_exact") else "—", rl, ma))


if __name__ == "__main__":
    sys.path.insert(0, ".")
    main(sys.argv[1], sys.argv[2])
