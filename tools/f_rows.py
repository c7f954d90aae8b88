"""Timings of the SURVEY 8(f) kernels at the headline shape (768x1408, 12 heads, d=128, W=4):
frame_mass_kernel (scored eviction) and token_mask_kernel (segment / causal masks, 2 frames).
CUDA events around N back-to-back launches on the current stream; writes profiles/r1_f_rows.json.

    python tools/f_rows.py [--out FILE]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import paper_2510_12747_b200 as fv  # noqa: E402


def timed(fn, reps=50, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(os.path.dirname(HERE), "profiles", "r1_f_rows.json"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    rows, cols, heads, d, window, topk = 48, 88, 12, 128, 4, 27
    n = rows * cols
    gen = torch.Generator(device="cuda").manual_seed(3)
    rnd = lambda: torch.randn((heads, n, d), generator=gen, device="cuda").to(torch.bfloat16)
    ring = fv.KVRing(1, heads, d, rows, cols, window)
    for t in range(window + 1):
        ring.append(0, t, rnd(), rnd())
        if t < window:
            ring.evict(0)
    q = rnd()
    ring.attention(0, q, [window], fv.Mask.all_allowed(), topk)
    res = {"shape": "768x1408 latent (48x88), 12 heads, d=128, W=4 (5 frames, 198 key blocks), top-k 27"}
    us = timed(lambda: ring.frame_mass(0, [window], check_errors=False))
    res["frame_mass"] = {"avg_us": us, "note": "per layer-step, all 12 heads; includes the Python/C-ABI call "
                                               "(launch-bound loop)"}
    L = 2 * n
    seg = np.random.default_rng(0).permutation(np.arange(L) % 7).astype(np.int32)
    frame = np.repeat(np.arange(2), n).astype(np.int32)
    words = L * ((L + 63) // 64) * 8
    for name, fn in (("segment_mask", lambda: fv.build_segment_mask(seg)),
                     ("causal_mask", lambda: fv.build_causal_mask(frame, 0))):
        us = timed(fn, reps=20)
        res[name] = {"L": L, "bytes_written": words, "avg_us": us, "gbs": words / (us * 1e-6) / 1e9,
                     "note": "includes host label validation, the label H2D copy and the output allocation"}
    print(json.dumps(res, indent=1))
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
