#!/usr/bin/env python
"""One configs.py point (for ncu launch lists of a single config).

    python tools/point.py ROWS COLS TOPK [loc EH EW trunc|pres] [--steps N]
"""
import argparse
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import paper_2510_12747_b200 as fv  # noqa: E402
from configs import run_point  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("rows", type=int)
ap.add_argument("cols", type=int)
ap.add_argument("topk", type=int)
ap.add_argument("mask", nargs="*")
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--heads", type=int, default=12)
a = ap.parse_args()
m = fv.Mask.all_allowed()
if a.mask and a.mask[0] == "loc":
    m = fv.Mask.locality(int(a.mask[1]), int(a.mask[2]), truncated=a.mask[3] == "trunc")
ctx = fv.Context.default()
ctx.read_tiles()
r = run_point(a.rows, a.cols, a.heads, 128, 4, a.topk, m, layers=2, steps=a.steps, warmup=2)
tiles, full = ctx.read_tiles()
r["tiles_per_step"] = tiles / (2 * a.steps + 2)  # timed loop + span pass + warm-up steps
r["full_tiles_per_step"] = full / (2 * a.steps + 2)
print(r)
