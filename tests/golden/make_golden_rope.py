"""Regenerate tests/golden/rope.npz from the UNMODIFIED reference (oracle/_ref).

    python tests/golden/make_golden_rope.py

apply_rope (P/src/rope.cpp:30-62) at TokenGrid positions for seeded vsr::Rng inputs,
bf16-rounded first (what the fused GPU path consumes): default split and a custom split,
frame ids past 0 so the temporal axis rotates.  Stored as raw fp32 bits."""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402  (test infrastructure)

# name, seed, d, frame ids, rows, cols, theta0, axis split
CASES = [
    ("d64_f3", 31, 64, [3], 8, 16, 10000.0, None),
    ("d128_two", 32, 128, [6, 7], 16, 24, 10000.0, None),
    ("d64_split", 33, 64, [41], 12, 20, 500.0, [16, 32, 16]),
]


def main():
    ref = oracle.Ref()
    arrays, meta = {}, []
    for name, seed, d, fids, rows, cols, theta0, split in CASES:
        L = len(fids) * rows * cols
        x = oracle.bf16_round(ref.gaussian(seed, L * d).reshape(L, d))
        arrays[name] = ref.apply_rope(x, fids, rows, cols, theta0, split)
        meta.append(dict(name=name, seed=seed, d=d, fids=fids, rows=rows, cols=cols, theta0=theta0, split=split))
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "rope.npz"), **arrays)
    print("wrote", os.path.join(HERE, "rope.npz"))


if __name__ == "__main__":
    main()
