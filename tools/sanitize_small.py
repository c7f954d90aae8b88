"""A small ring step (append + front + attention) and a plan/exec, for compute-sanitizer runs:

    compute-sanitizer --tool memcheck python tools/sanitize_small.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_12747_b200 as fv  # noqa: E402

torch.manual_seed(0)
heads, rows, cols, d = 2, 16, 24, 128
n = rows * cols
ring = fv.KVRing(1, heads, d, rows, cols, 2)
for t in range(4):
    q, k, v = [torch.randn((heads, n, d), device="cuda").to(torch.bfloat16) for _ in range(3)]
    out = ring.step(0, t, k, v, q, [t], fv.Mask.locality(9, 13, truncated=True), 3)
    ring.evict(0)
torch.cuda.synchronize()
fv.Context.default().check_errors()
print("ok", float(out.float().abs().sum()))
